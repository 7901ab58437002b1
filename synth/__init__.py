"""Seeded synthetic inputs shared by tests, bench and oracle tests (no method arithmetic)."""
from . import rng, configs  # noqa: F401
