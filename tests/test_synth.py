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


def test_planner_spec_instance():
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_planner_instance.json")))
    a, b, obj = planner.greedy(g["p"], g["m"], g["N"], g["rho"], g["M"])
    assert a == g["alpha"] and b == g["beta"] and abs(obj - g["objective"]) < 1e-12
    a2, b2, obj2 = planner.brute_force(g["p"], g["m"], g["N"], g["rho"], g["M"])
    assert abs(obj2 - g["objective"]) < 1e-12


def test_planner_marginal_gain_examples():
    """SPEC S:379-381 examples."""
    st = planner.marginal_gains(10, 4, 3, 0.25)
    assert [(round(t, 12), dm) for t, dm, _ in st] == [(3.5, 2.0), (1.5, 2.0)]
    st = planner.marginal_gains(1, 4, 3, 0.25)
    assert [(t, dm) for t, dm, _ in st] == [(0.25, 4)]


def test_planner_feasible_and_survey_counterexample():
    """one request p=1.4, m=16, N=3, rho=0.0202, M=11.93 -> hidden is optimal."""
    a, b, obj = planner.greedy([1.4], [16.0], 3, 0.0202, 11.93)
    assert a == [1] and b == [1] and obj > 0
    rs = np.random.default_rng(0)
    for _ in range(200):
        n = int(rs.integers(1, 7))
        p = list(rs.uniform(0, 10, n))
        m = [float(2 * rs.integers(1, 11)) for _ in range(n)]
        M = float(rs.uniform(0, sum(m)))
        a, b, obj = planner.greedy(p, m, 10, 0.05, M)
        used = sum(mi * (1 - bi / 2) for mi, ai, bi in zip(m, a, b) if ai)
        assert used <= M + 1e-9
        assert obj <= planner.brute_force(p, m, 10, 0.05, M)[2] + 1e-9
