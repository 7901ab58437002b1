"""Pins the reference pool semantics (oracle/pool_oracle.py) to the paper's Fig. 6 and
SPEC.md's memory-pool contract; plus a fuzz of the SPEC invariants."""
import json
import os
import random

from oracle.pool_oracle import HIDDEN, KV, PoolOracle, blocks_needed

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_fig6_block_counts():
    g = json.load(open(os.path.join(GOLDEN, "fig6_pool.json")))
    p = PoolOracle(g["num_blocks"], g["block_size"])
    for r in g["requests"]:
        assert blocks_needed(r["tokens"], r["mode"], g["block_size"]) == r["blocks"]
        assert p.append([r["id"]], [r["mode"]], [r["tokens"]]) == "ok"
        assert sum(len(t) for t in p.table(r["id"])) == r["blocks"]
        assert all(len(t) == r["per_kind"] for t in p.table(r["id"]))
    assert p.num_free() == g["free_after"]
    # paper's illustrative ids have the same counts per kind (only counts bind)
    assert len(g["paper_ids"]["A_K"]) == len(p.table(0)[0])
    assert len(g["paper_ids"]["B_X"]) == len(p.table(1)[0])
    assert p.free_req(0) == 6


def test_hidden_is_half_of_kv():
    """P:269 'half the storage space'."""
    for n in range(0, 200, 7):
        for B in (1, 4, 16):
            assert blocks_needed(n, KV, B) == 2 * blocks_needed(n, HIDDEN, B)


def test_extend_arithmetic():
    """hidden 14 tokens, B=4: +2 -> 0 new blocks, +3 -> 1; KV 11: +1 -> 0."""
    p = PoolOracle(32, 4)
    assert p.append([1], [HIDDEN], [14]) == "ok"
    f = p.num_free()
    assert p.append([1], [HIDDEN], [2]) == "ok" and p.num_free() == f
    p2 = PoolOracle(32, 4)
    p2.append([1], [HIDDEN], [14])
    f = p2.num_free()
    assert p2.append([1], [HIDDEN], [3]) == "ok" and p2.num_free() == f - 1
    p3 = PoolOracle(32, 4)
    p3.append([2], [KV], [11])
    f = p3.num_free()
    assert p3.append([2], [KV], [1]) == "ok" and p3.num_free() == f


def test_oom_is_all_or_nothing_and_kv_needs_two():
    """OOM leaves the pool unchanged; 1 free block, KV 1 token -> OOM."""
    p = PoolOracle(5, 4)
    assert p.append([1], [HIDDEN], [16]) == "ok"   # 4 blocks
    snap = (list(p.free), dict(p.req))
    assert p.append([2], [KV], [1]) == "oom"
    assert (list(p.free), dict(p.req)) == snap
    # batch OOM: the first request alone would fit, the batch does not
    assert p.append([3, 4], [HIDDEN, HIDDEN], [4, 4]) == "oom"
    assert 3 not in p.req and p.num_free() == 1


def test_free_idempotent_and_lowest_id_first():
    p = PoolOracle(8, 2)
    assert p.append([7], [KV], [3]) == "ok"
    assert p.table(7) == ([0, 2], [1, 3])          # interleaved K then V per logical block
    assert p.free_req(7) == 4 and p.free_req(7) == 0
    assert p.append([8], [HIDDEN], [1]) == "ok" and p.table(8) == ([0],)


def test_mode_mismatch_and_duplicates():
    p = PoolOracle(8, 2)
    p.append([1], [KV], [1])
    assert p.append([1], [HIDDEN], [1]) == "mode_mismatch"
    assert p.append([2, 2], [KV, KV], [1, 1]) == "invalid"


def test_bulk_equals_token_by_token():
    """For one request, a bulk append lays blocks out exactly as token-by-token appends."""
    for mode in (KV, HIDDEN):
        a, b = PoolOracle(64, 4), PoolOracle(64, 4)
        a.append([1], [mode], [13])
        for _ in range(13):
            b.append([1], [mode], [1])
        assert a.table(1) == b.table(1)


def test_fuzz_invariants():
    """conservation, no aliasing, K/V symmetry, fragmentation bound; 10^4 ops."""
    rs = random.Random(0)
    p = PoolOracle(97, 4)
    for _ in range(10_000):
        op = rs.random()
        if op < 0.6:
            k = rs.randint(1, 3)
            ids = rs.sample(range(30), k)
            modes = [p.req[i]["mode"] if i in p.req else rs.randint(0, 1) for i in ids]
            p.append(ids, modes, [rs.randint(0, 9) for _ in ids])
        else:
            p.free_req(rs.randrange(30))
        owned = [b for r in p.req.values() for b in r["K"] + r["V"] + r["X"]]
        assert len(owned) == len(set(owned))
        assert len(owned) + p.num_free() == 97
        assert not (set(owned) & set(p.free))
        for r in p.req.values():
            if r["mode"] == KV:
                assert len(r["K"]) == len(r["V"]) == -(-r["n"] // 4)
            else:
                assert len(r["X"]) == -(-r["n"] // 4) and not r["K"]
