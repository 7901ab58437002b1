"""Seeded generators: determinism, counter-offset consistency, distribution, planner fixture."""
import json
import os

import numpy as np
import torch

from synth import configs as C
from synth import planner, rng


def test_mix32_is_bijective_on_a_slice():
    x = torch.arange(0, 1 << 16, dtype=torch.int64) * 65521
    h = rng.mix32(x)
    assert h.unique().numel() == x.numel()
    assert int(h.max()) < 2 ** 32 and int(h.min()) >= 0


def test_normal_tensor_deterministic_and_offsets_consistent():
    a = rng.normal_tensor(5, rng.STREAM_X, 3, [40, 16], 1.0)
    b = rng.normal_tensor(5, rng.STREAM_X, 3, [40, 16], 1.0)
    assert torch.equal(a, b)
    part = rng.normal_tensor(5, rng.STREAM_X, 3, [10, 16], 1.0, offset=20 * 16)
    assert torch.equal(part, a[20:30])
    other = rng.normal_tensor(5, rng.STREAM_X, 4, [40, 16], 1.0)
    assert not torch.equal(a, other)


def test_normal_tensor_moments():
    z = rng.normal_tensor(1, rng.STREAM_Q, 0, [200_000], 1.0, torch.float32)
    assert abs(float(z.mean())) < 0.01 and abs(float(z.std()) - 1.0) < 0.01
    w = rng.normal_tensor(1, rng.STREAM_W, 0, [100_000], 0.1, torch.bfloat16)
    assert abs(float(w.float().std()) - 0.1) < 0.002


def test_workload_row_ranges_match_full():
    w = C.tiny()
    X = w.x(2)
    assert torch.equal(w.x(2, rows=(5, 17)), X[5:17])
    K, V = w.kv(0)
    K2, V2 = w.kv(0, rows=(16, 48))
    assert torch.equal(K2, K[16:48]) and torch.equal(V2, V[16:48])
    W = w.w_kv()
    assert torch.equal(w.w_kv(rows=(10, 40)), W[10:40])


def test_config_recipes():
    t = C.tiny()
    assert t.n == [64, 1, 33, 16] and t.modes == [0, 0, 1, 1]
    c4 = C.cfg4()
    assert len(c4.n) == 256 and min(c4.n) >= 32 and max(c4.n) <= 4096 and sum(c4.modes) == 128
    c2 = C.cfg2()
    assert len(c2.n) == 64 and max(c2.n) <= 2048 and sum(c2.modes) == 32
    hs = [sum(C.cfg5(h).modes) for h in C.CFG5_FRACTIONS]
    assert hs == sorted(hs) and hs[0] == 0 and hs[-1] == 256
    # nested prefixes of one permutation
    a, b = C.cfg5(1 / 8).modes, C.cfg5(1 / 4).modes
    assert all(y >= x for x, y in zip(a, b))


def test_cfg3_modes_are_the_oracle_planners_decision():
    """cfg3's cache modes come from the native planner (synth.planner delegates to
    hc_schedule); the oracle planner written from the paper (oracle/planner_oracle.py) takes
    the same decision on the same scenario — 127 of 128 candidates scheduled, 30 hidden."""
    from oracle import planner_oracle as PO
    from synth.configs import OPT30B, sharegpt_like
    rs = np.random.default_rng(2)
    n_all = sharegpt_like(128, rs)
    state = rs.bit_generator.state
    a, b = planner.plan_cfg3(n_all, OPT30B, rs)
    rs.bit_generator.state = state
    cfg, reqs, now = planner.cfg3_scenario(n_all, OPT30B, rs)
    a2, b2, _, res = PO.schedule(cfg, reqs, now)
    assert a == a2[:128] and b == b2[:128]
    assert sum(a) == 127 and sum(b) == 30 and res["iter_type"] == 0
    w = C.cfg3()
    assert w.req_ids == [i for i in range(128) if a[i]] and w.modes == [b[i] for i in range(128) if a[i]]
