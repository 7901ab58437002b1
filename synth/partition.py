"""Request sharding across GPUs; host logic only, no method arithmetic.

Weak scaling (the bench default): every rank runs its own full batch (configs.shard_for_rank).
Strong scaling: one batch split across ranks by LPT (longest processing time first) on the
roofline cost model: a KV token costs 2·d·s bytes at HBM bandwidth, a hidden token
4·d² FLOPs at tensor peak (plus its 2·d·s bytes of X).  Every rank computes the same
assignment from the global request list (deterministic tie-break by request index).
"""
from __future__ import annotations

import heapq
from typing import List, Sequence


def request_cost(n: int, mode: int, d: int, s: int = 2, bw: float = 6.5e12, flops: float = 1.4e15) -> float:
    if mode == 1:
        return n * (4.0 * d * d / flops + d * s / bw)
    return n * 2.0 * d * s / bw


def lpt(costs: Sequence[float], n_parts: int) -> List[List[int]]:
    """Assign items to n_parts bins, largest first, each to the currently lightest bin."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, p) for p in range(n_parts)]
    parts: List[List[int]] = [[] for _ in range(n_parts)]
    for i in order:
        load, p = heapq.heappop(heap)
        parts[p].append(i)
        heapq.heappush(heap, (load + costs[i], p))
    return [sorted(p) for p in parts]


def strong_shard(w, rank: int, world: int):
    """The rank's share of workload w under LPT (strong scaling)."""
    costs = [request_cost(n, m, w.shape.d, w.elem_bytes) for n, m in zip(w.n, w.modes)]
    idx = lpt(costs, world)[rank]
    return w.subset(idx, name=w.name)
