"""N>1 host logic on CPU with torch.distributed gloo, world_size 2: weak-scaling shards,
LPT strong sharding, and the bench's max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import configs as C
from synth import partition as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = C.shard_for_rank(C.cfg4(), rank, world)
    # every rank sees the same recipe sizes but its own request ids
    ids = torch.tensor(w.req_ids[:4], dtype=torch.int64)
    gathered = [torch.zeros_like(ids) for _ in range(world)]
    dist.all_gather(gathered, ids)
    # bench.py's timing rule: the step time is the MAX over ranks
    ms = torch.tensor([10.0 + 5.0 * rank])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # strong scaling: every rank derives the same LPT assignment independently
    parts = P.lpt([P.request_cost(n, m, 9216) for n, m in zip(w.n, w.modes)], world)
    mine = torch.tensor([len(parts[rank]), sum(w.n[i] for i in parts[rank])], dtype=torch.int64)
    all_parts = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(all_parts, mine)
    out[rank] = {"ids": [g.tolist() for g in gathered], "ms": float(ms.item()),
                 "n_tok": w.n_tokens(), "parts": [p.tolist() for p in all_parts]}
    dist.destroy_process_group()


def test_gloo_world2_sharding_and_max_timing():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    r0, r1 = out[0], out[1]
    assert r0["ms"] == r1["ms"] == 15.0
    assert r0["n_tok"] == r1["n_tok"]
    a, b = r0["ids"]
    assert set(a).isdisjoint(b)                      # distinct requests per rank
    assert r0["parts"] == r1["parts"]               # identical LPT on every rank
    assert sum(p[0] for p in r0["parts"]) == 256


def test_lpt_balance_and_coverage():
    w = C.cfg4()
    costs = [P.request_cost(n, m, w.shape.d) for n, m in zip(w.n, w.modes)]
    for G in (2, 4, 8):
        parts = P.lpt(costs, G)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(costs)))
        loads = [sum(costs[i] for i in p) for p in parts]
        assert max(loads) / (sum(loads) / G) < 1.05     # near-linear strong scaling possible
    # LPT bound (4/3 - 1/(3G)) on a classic instance
    parts = P.lpt([3, 3, 2, 2, 2], 2)
    assert sorted(sum([3, 3, 2, 2, 2][i] for i in p) for p in parts) == [5, 7]


def test_strong_shard_subsets_partition_the_batch():
    w = C.cfg2()
    subs = [P.strong_shard(w, r, 4) for r in range(4)]
    ids = sorted(i for s in subs for i in s.req_ids)
    assert ids == sorted(w.req_ids)


def test_lpt_split_covers_every_token_once_and_balances():
    """Phase-2 plan: every request's tokens are covered exactly once, split parts sit on
    distinct ranks, ranges are block-aligned, and one dominant hidden request no longer
    bounds the makespan (cfg5 at 1/64 hidden on 8 ranks)."""
    w = C.cfg5(1 / 64)
    d, B = w.shape.d, w.block_size
    costs = [P.request_cost(n, m, d) for n, m in zip(w.n, w.modes)]
    for G in (2, 4, 8):
        plan = P.lpt_split(w.n, w.modes, d, G, B)
        cover = {}
        for r, items in enumerate(plan):
            held = [i for i, _, _ in items]
            assert len(held) == len(set(held))           # parts of one request on distinct ranks
            for i, t0, t1 in items:
                assert t0 % B == 0 and t0 < t1 <= w.n[i]
                cover.setdefault(i, []).append((t0, t1))
        for i, n in enumerate(w.n):
            rs = sorted(cover[i])
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        load = [sum(costs[i] * (t1 - t0) / w.n[i] for i, t0, t1 in items) for items in plan]
        ideal = sum(costs) / G
        unsplit = [sum(costs[i] for i in p) for p in P.lpt(costs, G)]
        assert max(load) <= max(unsplit) + 1e-12
        assert max(load) / ideal < 1.15


def _bench_dry(extra, world):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HC_BENCH_DRY="1", HC_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(world), "--steps", "3",
                        "--warmup", "3"] + extra, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout   # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("extra,scaling,total", [([], "strong", 256), (["--weak"], "weak", 4 * 256),
                                                 (["--no-gather"], "strong", 256)])
def test_bench_spawns_ranks_and_runs_its_multi_rank_control_path(extra, scaling, total):
    """`python bench.py --gpus 4` outside torchrun spawns 4 ranks itself (gloo here); cfg4 is
    strong-scaled by default (256 requests in total), --weak gives each rank a
    full batch; the output all-gather is on by default."""
    d = _bench_dry(extra, 4)
    assert d["n_gpus"] == 4 and d["scaling"] == scaling and d["config"]["n_req_total"] == total
    assert d["dry"] is True and d["ms_per_step"] > 0
    assert ("gloo all-gather" in d["config"]["output_gather"]) == ("--no-gather" not in extra)
