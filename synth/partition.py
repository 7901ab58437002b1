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


def lpt_split(ns: Sequence[int], modes: Sequence[int], d: int, world: int, block: int = 16, s: int = 2):
    """LPT with token-range splitting (SURVEY §8(e) phase 2).  A request whose cost exceeds
    the ideal per-rank load (total / world) is cut into k = ceil(cost / ideal) (<= world)
    block-aligned token ranges on k distinct ranks; their (out, lse) partials are merged
    by hc_merge_partials.  Everything else is plain LPT.  Returns, per rank, a list of
    (request index, token begin, token end); every rank derives the same plan."""
    costs = [request_cost(n, m, d, s) for n, m in zip(ns, modes)]
    ideal = sum(costs) / world
    items = []   # (cost, request, begin, end)
    for i, (n, c) in enumerate(zip(ns, costs)):
        k = min(world, max(1, int(-(-c // ideal)) if ideal > 0 else 1))
        nb = -(-n // block)
        k = min(k, nb)
        if k == 1:
            items.append((c, i, 0, n))
            continue
        # k block-aligned ranges with (almost) equal block counts
        b0 = 0
        for p in range(k):
            b1 = b0 + nb // k + (1 if p < nb % k else 0)
            t0, t1 = b0 * block, min(n, b1 * block)
            items.append((c * (t1 - t0) / n, i, t0, t1))
            b0 = b1
    order = sorted(range(len(items)), key=lambda j: (-items[j][0], items[j][1], items[j][2]))
    heap = [(0.0, p) for p in range(world)]
    plan: List[list] = [[] for _ in range(world)]
    for j in order:
        c, i, t0, t1 = items[j]
        # parts of one request go to distinct ranks: take the lightest rank not holding it
        popped = []
        while True:
            load, p = heapq.heappop(heap)
            if all(r != i for r, _, _ in plan[p]) or not heap:
                break
            popped.append((load, p))
        plan[p].append((i, t0, t1))
        heapq.heappush(heap, (load + c, p))
        for x in popped:
            heapq.heappush(heap, x)
    return [sorted(p) for p in plan]
