"""Reference semantics of Apt-Serve's adaptive scheduler (NEXT row f2).

TEST INFRASTRUCTURE ONLY (see oracle/hc_oracle.py header for who may import it).

Written step by step from PAPER.md §4.2 and §5, in the paper's
order and notation, with SPEC.md's tie-breaks where the paper is silent:

  runtime tracking      p_i = now - arrival (no output token yet) or now - last token
                                 m_i = KV memory of the sequence incl. this iteration's token
  SLO fallback   a violated request's p_i becomes eps (near-zero) or decay * p_i
  iteration type        prefill iff sum_W p > sum_R p (ties -> decode); U = W or R
  budget                M = M~ - sum_R m_i (prefill) or M~ (decode), clamped at 0
  values (Eq. 5-6)              g_i = p_i - beta_i (|W|+|R|) rho m_i
  marginal gains    theta = 2p/m - 2N rho (hidden, dm = m/2), 2N rho (upgrade, dm = m/2),
                                 refined to p/m (direct KV, dm = m) when p/m < 2N rho
  greedy over Upsilon (Eq. 10-11), theta desc / dm asc / index asc; then the best single
  feasible assignment (KV or hidden) if better (reading R14: the paper's
  refinement alone can schedule nothing when a hidden-only fit exists).
"""
from __future__ import annotations

import math
from typing import List, Sequence


def kv_units(tokens: int, block_size: int = 1) -> float:
    """KV memory of `tokens` tokens: a K and a V unit per block."""
    b = max(1, block_size)
    return 2.0 * math.ceil(tokens / b)


def pending_time(req: dict, now: float) -> float:
    """'current time minus the time it arrives' / 'minus the last time it has
    received an output token'."""
    t0 = req["last_token_time"] if req["has_token"] else req["arrival_time"]
    return max(0.0, now - t0)


def schedule(cfg: dict, reqs: Sequence[dict], now: float):
    """Returns (alpha, beta, g, result) for every input request (non-candidates 0)."""
    n = len(reqs)
    alpha, beta, g = [0] * n, [0] * n, [0.0] * n
    p = [pending_time(r, now) for r in reqs]
    m = [kv_units(r["seq_len"] + 1, cfg.get("block_size", 1)) for r in reqs]
    W = [i for i in range(n) if not reqs[i]["running"]]
    R = [i for i in range(n) if reqs[i]["running"]]
    if not W and not R:
        return alpha, beta, g, {"iter_type": -1, "n_candidates": 0, "budget": 0.0, "objective": 0.0,
                                "memory_used": 0.0}
    sum_w, sum_r = sum(p[i] for i in W), sum(p[i] for i in R)
    if not R:
        prefill = True
    elif not W:
        prefill = False
    else:
        prefill = sum_w > sum_r
    U = W if prefill else R
    M = max(0.0, cfg["total_units"] - sum(m[i] for i in R)) if prefill else cfg["total_units"]
    N = len(W) + len(R)
    rho = cfg["rho"]
    # SLO-aware fallback on the pending time of violated requests
    pc = {}
    for i in U:
        slo = cfg["tbt_slo"] if reqs[i]["has_token"] else cfg["ttft_slo"]
        pi = p[i]
        if slo > 0 and pi > slo:
            pi = cfg["decay"] * pi if cfg["fallback"] == 1 else cfg["eps"]
        pc[i] = pi

    def value(i, b):      # Eq. 5-6
        return pc[i] - b * N * rho * m[i]

    # Upsilon: (theta, r, dm, kind)
    ups = []
    for pos, i in enumerate(U):
        if m[i] <= 0:
            continue
        if cfg["hybrid"] and pc[i] / m[i] >= 2 * N * rho:
            ups.append((2 * pc[i] / m[i] - 2 * N * rho, m[i] / 2, pos, 0))   # hidden
            ups.append((2 * N * rho, m[i] / 2, pos, 1))                       # upgrade to KV
        else:
            ups.append((pc[i] / m[i], m[i], pos, 2))                          # refined: direct KV
    # ties: theta desc, delta-m asc, lower request id, stage order
    ups.sort(key=lambda s: (-s[0], s[1], reqs[U[s[2]]]["id"], s[2], s[3]))
    a = {i: 0 for i in U}
    b = {i: 0 for i in U}
    used = 0.0
    tol = 1e-9 * max(1.0, M)
    for theta, dm, pos, kind in ups:
        i = U[pos]
        if used + dm > M + tol:
            continue
        if kind == 0:
            a[i], b[i] = 1, 1
        elif kind == 1:
            if not (a[i] and b[i]):
                continue
            b[i] = 0
        else:
            a[i], b[i] = 1, 0
        used += dm
    obj = sum(value(i, b[i]) for i in U if a[i])
    best, best_ib = obj, None
    for i in U:
        for bb in ((0, 1) if cfg["hybrid"] else (0,)):
            if m[i] * (1 - bb / 2) <= M + tol and value(i, bb) > best:
                best, best_ib = value(i, bb), (i, bb)
    if best_ib is not None:
        a = {i: 0 for i in U}
        b = {i: 0 for i in U}
        a[best_ib[0]], b[best_ib[0]] = 1, best_ib[1]
        obj = best
    mem = 0.0
    for i in U:
        alpha[i], beta[i] = a[i], b[i]
        g[i] = value(i, b[i])
        if a[i]:
            mem += (1 - b[i] / 2) * m[i]
    return alpha, beta, g, {"iter_type": 1 if prefill else 0, "n_candidates": len(U), "budget": M,
                            "objective": obj, "memory_used": mem}


def brute_force(cfg: dict, reqs: Sequence[dict], now: float) -> float:
    """Definition 1 by exhaustive search over {skip, hidden, KV}^|U| (|U| <= 10)."""
    _, _, _, res = schedule(dict(cfg, hybrid=cfg["hybrid"]), reqs, now)
    n = len(reqs)
    p = [pending_time(r, now) for r in reqs]
    m = [kv_units(r["seq_len"] + 1, cfg.get("block_size", 1)) for r in reqs]
    W = [i for i in range(n) if not reqs[i]["running"]]
    R = [i for i in range(n) if reqs[i]["running"]]
    U = W if res["iter_type"] == 1 else R
    assert len(U) <= 10
    N = len(W) + len(R)
    M = res["budget"]
    pc = []
    for i in U:
        slo = cfg["tbt_slo"] if reqs[i]["has_token"] else cfg["ttft_slo"]
        pi = p[i]
        if slo > 0 and pi > slo:
            pi = cfg["decay"] * pi if cfg["fallback"] == 1 else cfg["eps"]
        pc.append(pi)
    best = 0.0
    for code in range(3 ** len(U)):
        c, used, obj = code, 0.0, 0.0
        for k, i in enumerate(U):
            s = c % 3
            c //= 3
            if s == 0:
                continue
            bb = 1 if s == 1 else 0
            if bb and not cfg["hybrid"]:
                used = math.inf
                break
            used += m[i] * (1 - bb / 2)
            obj += pc[k] - bb * N * cfg["rho"] * m[i]
        if used <= M + 1e-9 * max(1.0, M):
            best = max(best, obj)
    return best


def calibrate_rho(m: Sequence[float], t: Sequence[float]) -> float:
    """Least-squares slope through the origin (Eq. 6's linear model)."""
    mm = sum(x * x for x in m)
    if not m or mm == 0:
        raise ValueError("degenerate calibration samples")
    return sum(x * y for x, y in zip(m, t)) / mm
