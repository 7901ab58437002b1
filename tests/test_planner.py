"""Adaptive scheduler (NEXT row f2): the oracle pinned to the paper/SPEC examples and brute
force, and the native planner (hc_schedule through the C ABI) bit-exact against the oracle."""
import json
import os
import random
import time

import pytest

from oracle import planner_oracle as PO

BASE = {"rho": 0.25, "total_units": 6.0, "ttft_slo": 0.0, "tbt_slo": 0.0, "fallback": 0, "eps": 1e-6,
        "decay": 0.4, "hybrid": 1, "block_size": 1}


def _req(i, p, m_units, running=True, now=100.0):
    """A request whose pending time is p and whose KV units are m (block_size 1: m = 2 (L+1))."""
    return {"id": i, "running": int(running), "has_token": int(running), "arrival_time": now - p,
            "last_token_time": now - p, "seq_len": int(m_units // 2) - 1}


# ---------------------------------------------------------------- oracle pins
def test_spec_greedy_instance():
    """r1(p=10,m=4) r2(6,2) r3(8,4), N=3, rho=.25, M=6 -> objective 18."""
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_planner_instance.json")))
    reqs = [_req(i, p, m) for i, (p, m) in enumerate(zip(g["p"], g["m"]))]
    a, b, gv, res = PO.schedule(dict(BASE, rho=g["rho"], total_units=g["M"]), reqs, 100.0)
    assert a == g["alpha"] and b == g["beta"] and abs(res["objective"] - g["objective"]) < 1e-12
    assert res["iter_type"] == 0 and res["memory_used"] == 6.0
    assert abs(PO.brute_force(dict(BASE, rho=g["rho"], total_units=g["M"]), reqs, 100.0) - 18.0) < 1e-12


def test_value_and_theta_examples():
    """SPEC S:326-327 (Eq. 5): p=10, beta=1, N=5, rho=.001, m=100 -> g = 9.5;
    S:379-381: theta stages (3.5, 1.5) and refined p/m = 0.25."""
    reqs = [_req(0, 10.0, 100)] + [_req(k, 0.0, 2, running=False) for k in range(1, 5)]
    cfg = dict(BASE, rho=0.001, total_units=50.0)
    a, b, g, res = PO.schedule(cfg, reqs, 100.0)
    assert res["iter_type"] == 0                       # sum_R p = 10 > sum_W p = 0
    assert a[0] == 1 and b[0] == 1 and abs(g[0] - 9.5) < 1e-12


def test_iteration_type_and_budget():
    """P:345 / S:383-392: larger cumulative pending time wins, ties -> decode; P:359 budget."""
    now = 10.0
    w = {"id": 1, "running": 0, "has_token": 0, "arrival_time": 6.0, "last_token_time": 0.0, "seq_len": 9}
    r = {"id": 2, "running": 1, "has_token": 1, "arrival_time": 0.0, "last_token_time": 9.0, "seq_len": 19}
    _, _, _, res = PO.schedule(dict(BASE, total_units=100.0), [w, r], now)
    assert res["iter_type"] == 1 and res["budget"] == 100.0 - 40.0      # prefill: M~ - sum_R m
    r2 = dict(r, last_token_time=6.0)                                   # tie: 4 = 4 -> decode
    _, _, _, res = PO.schedule(dict(BASE, total_units=100.0), [w, r2], now)
    assert res["iter_type"] == 0 and res["budget"] == 100.0
    _, _, _, res = PO.schedule(dict(BASE, total_units=30.0), [w, r], now)
    assert res["budget"] == 0.0                                         # clamped at 0
    _, _, _, res = PO.schedule(BASE, [], now)
    assert res["iter_type"] == -1


def test_slo_fallback_near_zero_and_decay():
    """P:314 near-zero demotion; P:584 decay factor 0.4."""
    late = {"id": 1, "running": 0, "has_token": 0, "arrival_time": 0.0, "last_token_time": 0.0, "seq_len": 1}
    ok = {"id": 2, "running": 0, "has_token": 0, "arrival_time": 9.5, "last_token_time": 0.0, "seq_len": 1}
    cfg = dict(BASE, total_units=2.0, ttft_slo=1.0, rho=0.0)   # one hidden slot (m/2 = 2)
    a, b, g, _ = PO.schedule(cfg, [late, ok], 10.0)
    assert abs(g[0] - 1e-6) < 1e-15 and a == [0, 1]            # only one fits; the violated one loses
    a, b, g, _ = PO.schedule(dict(cfg, fallback=1), [late, ok], 10.0)
    assert abs(g[0] - 4.0) < 1e-12 and a == [1, 0]            # decayed 0.4 * 10 = 4 > 0.5


def test_hidden_only_fit_is_scheduled():
    """SURVEY §4.3 counterexample: p=1.4, m=16, N=3, rho=.0202, M=11.93 -> hidden (refinement
    alone would schedule nothing)."""
    reqs = [_req(0, 1.4, 16)] + [_req(k, 0.0, 2, running=False) for k in (1, 2)]
    a, b, g, res = PO.schedule(dict(BASE, rho=0.0202, total_units=11.93), reqs, 100.0)
    assert a[0] == 1 and b[0] == 1 and res["objective"] > 0


def test_kv_only_ablation_uniform_m_is_optimal():
    """SPEC S:415 exactness escape: hybrid off and equal m -> greedy equals brute force."""
    rs = random.Random(3)
    for _ in range(100):
        n = rs.randint(1, 7)
        reqs = [_req(i, rs.uniform(0, 10), 8) for i in range(n)]
        cfg = dict(BASE, hybrid=0, total_units=float(8 * rs.randint(0, n)))
        _, _, _, res = PO.schedule(cfg, reqs, 100.0)
        assert abs(res["objective"] - PO.brute_force(cfg, reqs, 100.0)) < 1e-9


def test_feasibility_and_bounded_by_optimum_fuzz():
    rs = random.Random(4)
    for _ in range(300):
        n = rs.randint(1, 7)
        reqs = [_req(i, rs.uniform(0, 10), 2 * rs.randint(1, 10)) for i in range(n)]
        cfg = dict(BASE, rho=rs.uniform(0, 0.1), total_units=rs.uniform(0, 60))
        a, b, g, res = PO.schedule(cfg, reqs, 100.0)
        assert res["memory_used"] <= res["budget"] + 1e-9
        assert all(ai or not bi for ai, bi in zip(a, b))
        assert res["objective"] <= PO.brute_force(cfg, reqs, 100.0) + 1e-9


def test_calibrate_rho_examples():
    """{(1,.003),(2,.006)} -> .003; zeros -> 0."""
    assert abs(PO.calibrate_rho([1, 2], [0.003, 0.006]) - 0.003) < 1e-15
    assert PO.calibrate_rho([1, 2], [0.0, 0.0]) == 0.0
    with pytest.raises(ValueError):
        PO.calibrate_rho([0, 0], [1, 1])


# ---------------------------------------------------------------- native planner via the ABI
@pytest.fixture(scope="module")
def lib():
    from paper_2504_07494_b200 import build
    build.build()
    from paper_2504_07494_b200 import hc
    return hc


def native_schedule(hc, cfg, reqs, now):
    a, b, g, res = hc.schedule(cfg, reqs, now)

    class R:
        pass
    r = R()
    r.__dict__.update(res)
    return a, b, g, r


def test_native_planner_matches_oracle(lib):
    """Bit-exact decisions (alpha, beta) and values on random mixed W/R instances with SLOs,
    both fallback modes, hybrid on/off and several block sizes."""
    rs = random.Random(5)
    for trial in range(400):
        n = rs.randint(0, 40)
        now = 1000.0
        reqs = []
        for i in range(n):
            running = rs.random() < 0.5
            has = running or rs.random() < 0.2
            reqs.append({"id": i, "running": int(running), "has_token": int(has),
                         "arrival_time": now - rs.uniform(0, 5), "last_token_time": now - rs.uniform(0, 1),
                         "seq_len": rs.randint(0, 3000)})
        cfg = {"rho": rs.choice([0.0, 1e-6, 4.57e-8 * 80, rs.uniform(0, 1e-4)]),
               "total_units": rs.uniform(0, 60000), "ttft_slo": rs.choice([0.0, 1.5, 3.0]),
               "tbt_slo": rs.choice([0.0, 0.2, 0.5]), "fallback": rs.randint(0, 1), "eps": 1e-6, "decay": 0.4,
               "hybrid": rs.randint(0, 1), "block_size": rs.choice([1, 4, 16])}
        a, b, g, res = native_schedule(lib, cfg, reqs, now)
        a2, b2, g2, res2 = PO.schedule(cfg, reqs, now)
        assert (a, b) == (a2, b2), trial
        assert res.iter_type == res2["iter_type"] and res.n_candidates == res2["n_candidates"]
        assert abs(res.objective - res2["objective"]) <= 1e-9 * max(1.0, abs(res2["objective"]))
        assert all(abs(x - y) <= 1e-9 * max(1.0, abs(y)) for x, y in zip(g, g2))


def test_native_calibrate_rho(lib):
    assert abs(lib.calibrate_rho([1.0, 2.0], [0.003, 0.006]) - 0.003) < 1e-15
    with pytest.raises(lib.HcError):
        lib.calibrate_rho([0.0, 0.0], [0.003, 0.006])


def test_native_planner_time_vs_candidates(lib):
    """Paper Table 6 reports 0.3 / 0.5 / 1.0 / 2.1 / 4.8 / 10.8 ms for 50 ... 1600
    candidates; the native planner must stay below those (it is O(n log n))."""
    paper_ms = {50: 0.3, 100: 0.5, 200: 1.0, 400: 2.1, 800: 4.8, 1600: 10.8}
    rs = random.Random(6)
    for n, ms in paper_ms.items():
        reqs = [{"id": i, "running": 1, "has_token": 1, "arrival_time": 0.0, "last_token_time": 999.0 - rs.random(),
                 "seq_len": rs.randint(1, 2000)} for i in range(n)]
        cfg = dict(BASE, rho=1e-6, total_units=1000.0 * n)
        t0 = time.perf_counter()
        for _ in range(20):
            native_schedule(lib, cfg, reqs, 1000.0)
        dt = (time.perf_counter() - t0) / 20 * 1e3
        assert dt < ms, (n, dt)


def test_greedy_ties_follow_request_id_not_input_order(lib):
    """SPEC S:376 / S:412: equal theta and delta-m -> the lower request id is accepted first, so
    the decision does not depend on the order requests are handed in (oracle and native)."""
    # four identical running requests (same p, same m); budget fits exactly two hidden stages
    reqs = [_req(i, 4.0, 8) for i in (7, 3, 9, 1)]
    cfg = dict(BASE, rho=0.01, total_units=8.0)
    for order in ([0, 1, 2, 3], [3, 2, 1, 0], [2, 0, 3, 1]):
        rr = [reqs[k] for k in order]
        for sched in (PO.schedule, lambda c, r, t: native_schedule(lib, c, r, t)):
            a, b, _, _ = sched(cfg, rr, 100.0)
            picked = sorted(r["id"] for r, x in zip(rr, a) if x)
            assert picked == [1, 3], (order, picked)
