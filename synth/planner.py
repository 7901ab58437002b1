"""cfg3's cache-mode assignment: the request mix comes from the adaptive
scheduler itself — the library's native planner `hc_schedule` (§5, P:349-390;
NEXT row f2, pinned bit-exact against oracle/planner_oracle.py in tests/test_planner.py).
This module only states the cfg3 scenario; it implements none of the planner.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def cfg3_scenario(n_ctx: List[int], shape, rs: np.random.Generator) -> Tuple[dict, list, float]:
    """One decode iteration of an OPT-30B server (SURVEY §8(d) cfg3 recipe):
    128 running candidates with pending time p_i ~ U(0, 1.5 s) (30B TTFT SLO) and KV
    need m_i = 2 (n_i + 1) units (block size 1), 64 waiting requests with no
    pending time (so N = |W| + |R| = 192 and the iteration is a decode iteration),
    rho = (4 d^2 / F) / 2 with F = 2.25e15 (ideal per-layer rebuild time per unit), and a
    budget of 0.75 * sum m.  Returns (sched config, requests, now) for hc_schedule."""
    p = [float(v) for v in rs.uniform(0.0, 1.5, size=len(n_ctx))]
    now = 1000.0
    reqs = [{"id": i, "running": 1, "has_token": 1, "arrival_time": 0.0, "last_token_time": now - p[i],
             "seq_len": int(n_ctx[i])} for i in range(len(n_ctx))]
    reqs += [{"id": len(n_ctx) + k, "running": 0, "has_token": 0, "arrival_time": now, "last_token_time": 0.0,
              "seq_len": 1} for k in range(64)]
    m = [2.0 * (n + 1) for n in n_ctx]
    cfg = {"rho": (4.0 * shape.d ** 2 / 2.25e15) / 2.0, "total_units": 0.75 * sum(m), "ttft_slo": 0.0,
           "tbt_slo": 0.0, "fallback": 0, "eps": 1e-6, "decay": 0.4, "hybrid": 1, "block_size": 1}
    return cfg, reqs, now


def plan_cfg3(n_ctx: List[int], shape, rs: np.random.Generator):
    """(alpha, beta) of the 128 candidates, decided by the native planner."""
    from paper_2504_07494_b200 import hc
    cfg, reqs, now = cfg3_scenario(n_ctx, shape, rs)
    alpha, beta, _, _ = hc.schedule(cfg, reqs, now)
    k = len(n_ctx)
    return [int(a) for a in alpha[:k]], [int(b) for b in beta[:k]]
