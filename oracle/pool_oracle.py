"""Reference semantics of the unified block pool.

TEST INFRASTRUCTURE ONLY (see oracle/hc_oracle.py header for who may import it).

PAPER.md §4.3: one global pool of fixed-size blocks; each block stores
K, V *or* X vectors for B consecutive token positions of one request; blocks of a
request need not be contiguous; blocks are chosen "by scanning the available unused
cache blocks".  Block accounting follows SPEC.md domain-core:
KV -> 2*ceil(n/B) unit blocks (a K list and a V list), hidden -> ceil(n/B).
Pool contract (SPEC.md memory-pool S:163-219): lowest-id-first, all-or-nothing
over a whole append call, extend allocates only when the last block is
full, free returns the count and is idempotent, K/V lists
symmetric.  Order within a KV request (reading R10): for each new logical
block, K takes the lowest free id, then V the next lowest; requests are served in
call order.  This makes a bulk append identical to token-by-token appends.
"""
from __future__ import annotations

import heapq
from typing import Dict, List, Sequence

KV, HIDDEN = 0, 1


def blocks_needed(n: int, mode: int, B: int) -> int:
    """SPEC S:58-66 (Fig. 6)."""
    per_kind = -(-n // B)
    return 2 * per_kind if mode == KV else per_kind


class PoolOracle:
    def __init__(self, num_blocks: int, B: int):
        self.num_blocks, self.B = num_blocks, B
        self.free: List[int] = list(range(num_blocks))
        heapq.heapify(self.free)
        self.req: Dict[int, dict] = {}

    def num_free(self) -> int:
        return len(self.free)

    def append(self, req_ids: Sequence[int], modes: Sequence[int], n_tokens: Sequence[int]):
        """All-or-nothing batch append.  Returns 'ok' | 'oom' | 'mode_mismatch' | 'invalid'."""
        if len(set(req_ids)) != len(req_ids):
            return "invalid"
        need = 0
        for r, m, t in zip(req_ids, modes, n_tokens):
            if t < 0 or m not in (KV, HIDDEN):
                return "invalid"
            cur = self.req.get(r)
            n0 = 0
            if cur is not None:
                if cur["mode"] != m:
                    return "mode_mismatch"
                n0 = cur["n"]
            need += blocks_needed(n0 + t, m, self.B) - blocks_needed(n0, m, self.B)
        if need > len(self.free):
            return "oom"
        for r, m, t in zip(req_ids, modes, n_tokens):
            cur = self.req.setdefault(r, {"mode": m, "n": 0, "K": [], "V": [], "X": []})
            new_lb = -(-(cur["n"] + t) // self.B) - -(-cur["n"] // self.B)
            for _ in range(new_lb):
                if m == KV:
                    cur["K"].append(heapq.heappop(self.free))
                    cur["V"].append(heapq.heappop(self.free))
                else:
                    cur["X"].append(heapq.heappop(self.free))
            cur["n"] += t
        return "ok"

    def free_req(self, r: int) -> int:
        cur = self.req.pop(r, None)
        if cur is None:
            return 0
        blocks = cur["K"] + cur["V"] + cur["X"]
        for b in blocks:
            heapq.heappush(self.free, b)
        return len(blocks)

    def table(self, r: int):
        c = self.req[r]
        return (c["K"], c["V"]) if c["mode"] == KV else (c["X"],)
