"""fp64 CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product (paper_2504_07494_b200/) never does.
"""
from . import hc_oracle, pool_oracle  # noqa: F401
