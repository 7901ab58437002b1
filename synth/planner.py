"""Host-side greedy cache-mode planner (bench-input generator for cfg3; NEXT-f2 in full).

Follows PAPER.md §5: the value of scheduling request i is
    g_i = p_i - beta_i * (|W|+|R|) * t_i,   t_i = rho * m_i          (Eq. 5-6)
subject to  sum_i (1 - beta_i/2) m_i alpha_i <= M                    (Eq. 7)
solved greedily by marginal gain per memory unit theta, with SPEC.md's
tie-break and best-single comparison.  SURVEY.md §4.3 found that the paper's
refinement ("if p/m < 2N rho, hidden usage is avoided") drops feasible positive-value
hidden options; the best-single step here therefore also considers the hidden
assignment (reading R9).  This module produces beta only; it is not on the
GPU hot path and not an optimisation target (north_star).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

HIDDEN, UPGRADE, DIRECT = 0, 1, 2


def marginal_gains(p: float, m: float, N: int, rho: float, hybrid: bool = True):
    """Stages per SPEC S:373-381 / P:363-381: list of (theta, delta_m, stage)."""
    if m <= 0:
        return []
    if hybrid and p / m >= 2 * N * rho:
        return [(2 * p / m - 2 * N * rho, m / 2, HIDDEN), (2 * N * rho, m / 2, UPGRADE)]
    return [(p / m, m, DIRECT)]


def value(p: float, m: float, beta: int, N: int, rho: float) -> float:
    """Eq. 5-6."""
    return p - beta * N * rho * m


def greedy(p: List[float], m: List[float], N: int, rho: float, M: float,
           hybrid: bool = True) -> Tuple[List[int], List[int], float]:
    cands = []
    for i in range(len(p)):
        for th, dm, st in marginal_gains(p[i], m[i], N, rho, hybrid):
            cands.append((-th, dm, i, st))
    cands.sort()
    alpha = [0] * len(p)
    beta = [0] * len(p)
    used = 0.0
    hidden_taken = set()
    for _, dm, i, st in cands:
        if used + dm > M + 1e-12:
            continue
        if st == HIDDEN:
            alpha[i], beta[i] = 1, 1
            hidden_taken.add(i)
        elif st == UPGRADE:
            if i not in hidden_taken:
                continue
            beta[i] = 0
        else:
            alpha[i], beta[i] = 1, 0
        used += dm
    obj = sum(value(p[i], m[i], beta[i], N, rho) for i in range(len(p)) if alpha[i])
    # best single item, KV or hidden (SURVEY §4.3 fix)
    best, best_ab = obj, None
    for i in range(len(p)):
        for b in ((0, 1) if hybrid else (0,)):
            need = m[i] * (1 - b / 2)
            if need <= M + 1e-12:
                g = value(p[i], m[i], b, N, rho)
                if g > best:
                    best, best_ab = g, (i, b)
    if best_ab is not None:
        alpha = [0] * len(p)
        beta = [0] * len(p)
        alpha[best_ab[0]], beta[best_ab[0]] = 1, best_ab[1]
        obj = best
    return alpha, beta, obj


def brute_force(p, m, N, rho, M, hybrid=True):
    """Exhaustive 3^n search over {skip, hidden, KV}; n <= 12."""
    n = len(p)
    assert n <= 12
    best, best_ab = 0.0, ([0] * n, [0] * n)
    for code in range(3 ** n):
        a, b, used, obj, c = [0] * n, [0] * n, 0.0, 0.0, code
        for i in range(n):
            s = c % 3
            c //= 3
            if s == 0:
                continue
            if s == 1 and not hybrid:
                used = float("inf")
                break
            a[i], b[i] = 1, 1 if s == 1 else 0
            used += m[i] * (1 - b[i] / 2)
            obj += value(p[i], m[i], b[i], N, rho)
        if used <= M + 1e-12 and obj > best + 1e-12:
            best, best_ab = obj, (a, b)
    return best_ab[0], best_ab[1], best


def plan_cfg3(n_ctx: List[int], shape, rs: np.random.Generator):
    """cfg3 recipe: p_i ~ U(0, 1.5 s) (30B TTFT SLO);
    m_i = 2(n_i+1) units; N = 128 + 64; rho = (4 d^2 / F)/2 with F = 2.25e15
    (per-layer ideal reconstruction time per memory unit); M = 0.75 * sum m."""
    p = [float(v) for v in rs.uniform(0.0, 1.5, size=len(n_ctx))]
    m = [2.0 * (n + 1) for n in n_ctx]
    N = len(n_ctx) + 64
    rho = (4.0 * shape.d ** 2 / 2.25e15) / 2.0
    M = 0.75 * sum(m)
    alpha, beta, _ = greedy(p, m, N, rho, M)
    return alpha, beta
