"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same
seeded inputs.  Tolerances (BASELINE.json north_star): max normwise relative error
<= 1e-5 in fp32 mode, <= 1e-2 in bf16 (reading R12)."""
import math

import numpy as np
import pytest
import torch

from synth import configs as C
from synth.configs import MODE_HIDDEN, MODE_KV, LayerShape, Workload
from tests import hc_testlib as T

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5
TOL_BF16 = 1e-2
TOL_LSE = 1e-2          # absolute, natural log (lse of scores ~N(0,1): |lse| ~ ln n)


@pytest.fixture(scope="module")
def hc():
    from paper_2504_07494_b200 import build
    build.build()
    from paper_2504_07494_b200 import hc as m
    return m


def _run(w, flags=0, split_tokens=0, order="rr", idx=None):
    pool = T.make_pool(w, flags=flags, split_tokens=split_tokens)
    T.fill(pool, w, order=order)
    q = T.queries(w)
    out, lse = T.decode(pool, w, q, idx)
    return pool, out, lse


# ------------------------------------------------------------------ tiny fp32 (full)
@pytest.mark.parametrize("B", [16, 4])
@pytest.mark.parametrize("bias", [False, True])
def test_tiny_fp32_full(hc, B, bias):
    w = C.tiny(block_size=B, bias=bias)
    pool, out, lse = _run(w)
    err, lerr = T.compare(w, out, lse, range(4))
    assert err <= TOL_F32, err
    assert lerr <= 1e-5, lerr
    assert pool.last_launch_count() == 3  # reconstruction, attention, combine


def test_tiny_fp32_generic_attention_kernel(hc):
    w = C.tiny()
    _, out, lse = _run(w, flags=hc.HC_FLAG_GENERIC_ATTN)
    assert T.compare(w, out, lse, range(4))[0] <= TOL_F32


# ------------------------------------------------------------------ bf16, several tiles + ragged tails
SHAPES = [
    # (d, H, dh, B)
    (256, 2, 128, 16),
    (512, 8, 64, 32),
    (384, 3, 128, 8),     # B=8: generic attention, 16 TMA boxes per A tile
    (256, 2, 128, 64),
    (256, 2, 128, 256),   # block larger than an M tile
]
N_MIX = [1, 15, 16, 17, 129, 300, 513, 1000, 33, 2]


def _bf16_workload(d, H, dh, B, n=N_MIX, bias=False, seed=11, modes=None, Hk=0):
    shape = LayerShape(f"test-{d}" + (f"-gqa{Hk}" if Hk else ""), d, H, dh, Hk)
    if modes is None:
        modes = [MODE_KV if i % 2 == 0 else MODE_HIDDEN for i in range(len(n))]
    return Workload(f"bf16-{d}-{B}", shape, B, "bf16", seed, list(n), list(modes), list(range(len(n))), bias)


@pytest.mark.parametrize("d,H,dh,B", SHAPES)
def test_bf16_mixed_batch_vs_oracle(hc, d, H, dh, B):
    w = _bf16_workload(d, H, dh, B, bias=True)
    _, out, lse = _run(w)
    err, lerr = T.compare(w, out, lse, range(len(w.n)))
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE, lerr


@pytest.mark.parametrize("flags", ["simt", "generic"])
def test_bf16_alternative_kernels_agree(hc, flags):
    """The SIMT reconstruction and the generic attention kernel meet the same bar."""
    f = hc.HC_FLAG_FORCE_SIMT if flags == "simt" else hc.HC_FLAG_GENERIC_ATTN
    w = _bf16_workload(256, 2, 128, 16)
    _, out, lse = _run(w, flags=f)
    assert T.compare(w, out, lse, range(len(w.n)))[0] <= TOL_BF16


def test_bf16_all_hidden_many_tiles(hc):
    """M spans many 128-row tiles of the tcgen05 GEMM with a ragged last tile."""
    n = [700, 1, 333, 1025, 64, 65]
    w = _bf16_workload(512, 4, 128, 16, n=n, modes=[MODE_HIDDEN] * len(n), bias=True)
    _, out, lse = _run(w)
    assert T.compare(w, out, lse, range(len(n)))[0] <= TOL_BF16


# ------------------------------------------------------------------ invariants (north_star)
def test_constant_values_give_ones(hc):
    """V = 1 => out = 1 (softmax rows sum to 1).  Hidden: W_V = 0, b_V = 1 => V = 1."""
    d, H, dh, B = 256, 2, 128, 16
    w = _bf16_workload(d, H, dh, B, n=[5, 300, 17, 1000])
    dev = torch.device("cuda", 0)
    W = w.w_kv(device=dev)
    W[d:] = 0
    b = torch.zeros(2 * d, dtype=torch.float32, device=dev)
    b[d:] = 1.0
    pool = T.make_pool(w, w_kv=W, b_kv=b)
    data = {}
    for i in range(len(w.n)):
        if w.modes[i] == MODE_KV:
            K, _ = w.kv(i, device=dev)
            data[i] = (K, torch.ones_like(K))
        else:
            data[i] = w.x(i, device=dev)
    T.fill(pool, w, data=data)
    out, _ = T.decode(pool, w, T.queries(w))
    assert np.all(out == 1.0)


def test_single_token_returns_v1(hc):
    """n = 1 => out = v_1 exactly (KV); hidden => bf16(W_V x_1) up to reconstruction rounding."""
    w = _bf16_workload(256, 2, 128, 16, n=[1, 1])
    pool, out, lse = _run(w)
    K, V = w.kv(0)
    assert np.array_equal(out[0], V[0].float().numpy())
    assert T.compare(w, out[[1]], lse[[1]], [1])[0] <= TOL_BF16


@pytest.mark.parametrize("d", [256, 1024])
def test_block_placement_is_bitwise_irrelevant(hc, monkeypatch, d):
    """Same logical content, different physical blocks => bitwise-identical output.  'seq'
    fills give each request consecutive block ids; with HC_BLOCK_RUNS=1 the GEMM fetches runs of
    8 blocks as one 128-row TMA box (same smem image as 8 gathered 16-row boxes)."""
    n = [700, 33, 511, 1, 257, 96, 129, 64, 300, 17] if d == 1024 else N_MIX
    w = _bf16_workload(d, d // 128, 128, 16, n=n)
    _, a, la = _run(w, split_tokens=64, order="rr")
    _, b, lb = _run(w, split_tokens=64, order="seq")
    _, c, lc = _run(w, split_tokens=64, order="shuffle")
    monkeypatch.setenv("HC_BLOCK_RUNS", "1")
    _, e, le = _run(w, split_tokens=64, order="seq")
    assert np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(a, e)
    assert np.array_equal(la, lb) and np.array_equal(la, lc) and np.array_equal(la, le)
    assert T.compare(w, b, lb, range(len(w.n)))[0] <= TOL_BF16


@pytest.mark.parametrize("S", [16, 64, 512, 4096])
def test_split_size_invariance(hc, S):
    w = _bf16_workload(256, 2, 128, 16)
    _, out, lse = _run(w, split_tokens=S)
    assert T.compare(w, out, lse, range(len(w.n)))[0] <= TOL_BF16


def test_batch_invariance_and_determinism(hc):
    w = _bf16_workload(256, 2, 128, 16)
    pool = T.make_pool(w, split_tokens=64)
    T.fill(pool, w)
    q = T.queries(w)
    full, lf = T.decode(pool, w, q)
    again, la = T.decode(pool, w, q)
    assert np.array_equal(full, again) and np.array_equal(lf, la)
    for i in (0, 3, 6):
        alone, l1 = T.decode(pool, w, q, [i])
        assert np.array_equal(alone[0], full[i]) and np.array_equal(l1[0], lf[i])
    sub = [7, 2, 5]
    part, lp = T.decode(pool, w, q, sub)
    assert np.array_equal(part, full[sub])


def test_hidden_equals_kv_twin(hc):
    """hidden(X) == KV(K = bf16(X W_K^T + b_K), V = ...) (north_star invariant).
    The twin's K/V are the oracle's fp64 projections rounded to bf16 on the host."""
    from oracle import hc_oracle as O
    d, H, dh, B = 256, 2, 128, 16
    n = [40, 300, 7]
    w = _bf16_workload(d, H, dh, B, n=n, modes=[MODE_HIDDEN] * 3, bias=True)
    W, b = w.w_kv(), w.b_kv()
    twin = Workload("twin", w.shape, B, "bf16", w.seed, n, [MODE_KV] * 3, [100, 101, 102], True)
    dev = torch.device("cuda", 0)
    pool = T.make_pool(w, num_blocks=200)
    data_h, data_k = {}, {}
    for i in range(3):
        X = w.x(i)
        K, V = O.hidden_request_kv(X, W, b)
        data_h[i] = X.to(dev)
        data_k[i] = (torch.tensor(K).to(torch.bfloat16).to(dev), torch.tensor(V).to(torch.bfloat16).to(dev))
    T.fill(pool, w, data=data_h)
    T.fill(pool, twin, data=data_k)
    q = T.queries(w)
    oh, lh = pool.decode(w.req_ids, q, w.scale)
    ok, lk = pool.decode(twin.req_ids, q, w.scale)
    oh, ok = oh.float().cpu().numpy(), ok.float().cpu().numpy()
    assert O.max_rel_err(oh, ok, H) <= TOL_BF16
    assert np.abs(lh.cpu().numpy() - lk.cpu().numpy()).max() <= 2e-2


def test_switch_mode_by_free_and_reappend(hc):
    """Cache-type switch = discard + recompute: free, re-append in the other mode."""
    d, H, dh, B = 256, 2, 128, 16
    w = _bf16_workload(d, H, dh, B, n=[90, 31], modes=[MODE_KV, MODE_HIDDEN])
    pool = T.make_pool(w, num_blocks=64)
    T.fill(pool, w)
    with pytest.raises(hc.HcError) as e:
        pool.append([w.req_ids[0]], [MODE_HIDDEN], [1], x=w.x(0, device="cuda")[:1].contiguous())
    assert e.value.status == hc.HC_E_MODE_MISMATCH
    assert pool.free(w.req_ids[0]) == 2 * math.ceil(90 / B)
    w2 = _bf16_workload(d, H, dh, B, n=[90, 31], modes=[MODE_HIDDEN, MODE_HIDDEN])
    pool.append([w2.req_ids[0]], [MODE_HIDDEN], [90], x=w2.x(0, device="cuda"))
    out, lse = T.decode(pool, w2, T.queries(w2))
    assert T.compare(w2, out, lse, [0, 1])[0] <= TOL_BF16


def test_error_paths_on_device(hc):
    w = _bf16_workload(256, 2, 128, 16, n=[20, 20])
    pool = T.make_pool(w, num_blocks=16)
    T.fill(pool, w)
    q = T.queries(w)
    out, lse = pool.decode([], q[:0].contiguous(), 1.0)
    assert pool.last_launch_count() == 0
    for bad, code in (([0, 0], hc.HC_E_INVALID), ([0, 77], hc.HC_E_UNKNOWN_REQ)):
        with pytest.raises(hc.HcError) as e:
            hc.hc_decode_attention(pool.handle, bad, q, 1.0, torch.empty_like(q), None, pool.workspace([0]))
        assert e.value.status == code
    small = torch.empty(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(hc.HcError) as e:
        hc.hc_decode_attention(pool.handle, [0, 1], q, 1.0, torch.empty_like(q), None, small)
    assert e.value.status == hc.HC_E_WORKSPACE
    pool.append([5], [MODE_KV], [0])                # created with 0 tokens
    with pytest.raises(hc.HcError) as e:
        pool.decode([5], q[:1].contiguous(), 1.0)
    assert e.value.status == hc.HC_E_INVALID


# ------------------------------------------------------------------ OPT-shaped configs, sampled
def _sample(w, n_kv=4, n_hid=2):
    kv = [i for i in range(len(w.n)) if w.modes[i] == MODE_KV]
    hid = [i for i in range(len(w.n)) if w.modes[i] == MODE_HIDDEN]
    rs = np.random.default_rng(0)
    pick = list(rs.choice(kv, size=min(n_kv, len(kv)), replace=False)) if kv else []
    if hid:
        longest = max(hid, key=lambda i: w.n[i])
        others = [i for i in hid if i != longest]
        pick += [longest] + (list(rs.choice(others, size=min(n_hid - 1, len(others)), replace=False)) if others else [])
    return [int(i) for i in pick]


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4", "cfg5:0.015625", "cfg5:0.03125", "cfg5:1.0"])
def test_opt_shaped_sampled_parity(hc, cfg):
    """Full batch on the GPU in the bench's launch configuration (auto split, tcgen05
    GEMM, pipelined attention; cfg5 1/64 takes the KV-dominated <2,8,2> fused
    configuration, the others <3,5,2>); the oracle checks a seeded sample of requests
    (KV: all heads; hidden: 3 heads incl. the first and last) including the longest
    hidden one."""
    w = C.by_name(cfg)
    pool = T.make_pool(w)
    T.fill(pool, w)
    q = T.queries(w)
    out, lse = T.decode(pool, w, q)
    assert np.isfinite(out).all()
    idx = _sample(w)
    H = w.shape.H
    heads = {i: [0, H // 2, H - 1] for i in idx if w.modes[i] == MODE_HIDDEN}
    err, lerr = T.compare(w, out[idx], lse[idx], idx, heads)
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE, lerr


def test_synth_bit_identical_on_device():
    """The counter-based generator gives the same bits on CUDA and CPU, so the oracle can
    regenerate inputs on the host (no oracle input is read back from the GPU path)."""
    from synth import rng
    for dt in (torch.bfloat16, torch.float32):
        a = rng.normal_tensor(3, rng.STREAM_X, 17, [333, 96], 0.7, dt, "cpu", offset=12345)
        b = rng.normal_tensor(3, rng.STREAM_X, 17, [333, 96], 0.7, dt, "cuda", offset=12345).cpu()
        assert torch.equal(a, b)
    w = C.cfg4()
    assert torch.equal(w.w_kv(rows=(100, 140)), w.w_kv(device="cuda", rows=(100, 140)).cpu())


@pytest.mark.parametrize("env", [{"HC_FUSED": "0"}, {"HC_FUSED": "0", "HC_TC_1SM": "1"},
                                 {"HC_FUSED": "0", "HC_TC_NSUB": "1"}])
def test_bf16_alternative_gemm_schedules(hc, monkeypatch, env):
    """Non-default GEMM paths (stand-alone CTA-pair GEMM + attention kernel, the 1-SM
    tcgen05 kernel, 256-wide pair tiles) meet the same bar as the fused default."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = _bf16_workload(512, 4, 128, 16, bias=True)
    _, out, lse = _run(w)
    assert T.compare(w, out, lse, range(len(w.n)))[0] <= TOL_BF16


def test_fused_and_unfused_agree_bitwise(hc, monkeypatch):
    """The fused step kernel and the two-kernel path compute the same thing in the same
    order (same GEMM tiles, same split-K tasks) => identical bits."""
    w = _bf16_workload(512, 4, 128, 16, bias=True)
    _, a, la = _run(w, split_tokens=64)
    monkeypatch.setenv("HC_FUSED", "0")
    _, b, lb = _run(w, split_tokens=64)
    assert np.array_equal(a, b) and np.array_equal(la, lb)


@pytest.mark.parametrize("env", [{"HC_GROUP_N": "2"}, {"HC_GROUP_N": "3"}, {"HC_SYNC_W": "8"},
                                 {"HC_GROUP_N": "2", "HC_SYNC_W": "8"}, {"HC_GROUP_N": "-3"},
                                 {"HC_FUSED_CFG": "352"}, {"HC_FUSED_CFG": "282"}, {"HC_FUSED_CFG": "342"},
                                 {"HC_FUSED_CFG": "3424"}, {"HC_FUSED_CFG": "3224"},
                                 {"HC_DYN_TILES": "0"}, {"HC_DYN_TILES": "0", "HC_SYNC_W": "8"}])
def test_fused_schedules_agree_bitwise(hc, monkeypatch, env):
    """The fused kernel's raster (n-tiles per group, m-major groups), partner lockstep and
    configuration (GEMM stages, attention warps, extra epilogue warps that split a tile's
    heads) only reorder whole tiles / heads / KV tasks in time: every tile's k-order, every
    head's epilogue arithmetic and every KV task are unchanged => identical bits.  d=1024
    gives 4 n-tiles; 9 hidden requests give 7 m-tiles with a ragged last one."""
    n = [700, 33, 511, 1, 257, 96, 129, 64, 300, 17, 415, 640]
    modes = [MODE_HIDDEN if i % 4 != 1 else MODE_KV for i in range(len(n))]
    w = _bf16_workload(1024, 8, 128, 16, n=n, modes=modes, bias=True)
    _, a, la = _run(w, split_tokens=64)
    assert T.compare(w, a, la, range(len(n)))[0] <= TOL_BF16
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, b, lb = _run(w, split_tokens=64)
    assert np.array_equal(a, b) and np.array_equal(la, lb)


def test_cuda_graph_replay_bitwise(hc):
    """One decode call (descriptor upload from the runtime's pinned staging buffer + the
    fused kernel + combine) captured as a CUDA graph: replays equal the eager call bit for
    bit while the batch is fixed (bench.py's `cuda_graph` variant)."""
    from paper_2504_07494_b200 import hc as H
    n = [700, 33, 511, 1, 257, 96, 129, 64]
    modes = [MODE_HIDDEN if i % 3 != 1 else MODE_KV for i in range(len(n))]
    w = _bf16_workload(1024, 8, 128, 16, n=n, modes=modes, bias=True)
    pool = T.make_pool(w)
    T.fill(pool, w)
    q = T.queries(w)
    ids = list(w.req_ids)
    ws = pool.workspace(ids)
    out = torch.empty((len(n), w.shape.d), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((len(n), w.shape.H), dtype=torch.float32, device="cuda")
    H.hc_decode_attention(pool.handle, ids, q, w.scale, out, lse, ws, torch.cuda.current_stream())
    torch.cuda.synchronize()
    ref_out, ref_lse = out.clone(), lse.clone()
    out.zero_()
    lse.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        H.hc_decode_attention(pool.handle, ids, q, w.scale, out, lse, ws, torch.cuda.current_stream())
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref_out) and torch.equal(lse, ref_lse)


def test_cross_partition_merge_vs_oracle(hc):
    """SURVEY §8(e) phase 2: each request's tokens split into 3 partitions (stored as
    separate requests, as ranks holding part of a long request would), decoded
    separately, merged by hc_merge_partials == the oracle on the whole request.  A 4th
    partition that holds nothing (lse = -inf, out = NaN) must not change a bit."""
    from paper_2504_07494_b200 import hc as H
    n = [700, 300, 129, 1000, 40]
    modes = [MODE_HIDDEN, MODE_KV, MODE_HIDDEN, MODE_KV, MODE_HIDDEN]
    w = _bf16_workload(512, 4, 128, 16, n=n, modes=modes, bias=True)
    dev = torch.device("cuda", 0)
    data = {i: (w.kv(i, device=dev) if w.modes[i] == MODE_KV else w.x(i, device=dev)) for i in range(len(n))}
    cuts = {i: [0, 17, n[i] // 2, n[i]] for i in range(len(n))}
    pool = T.make_pool(w, num_blocks=T.pool_blocks(w) + 8 * len(n))
    q = T.queries(w)
    P, d, Hh = 3, w.shape.d, w.shape.H
    outs = torch.empty((P + 1, len(n), d), dtype=torch.bfloat16, device=dev)
    lses = torch.empty((P + 1, len(n), Hh), dtype=torch.float32, device=dev)
    for p in range(P):
        ids, toks, ks, vs, xs = [], [], [], [], []
        for i in range(len(n)):
            a, b = cuts[i][p], cuts[i][p + 1]
            ids.append(1000 * (p + 1) + i)
            toks.append(b - a)
            if w.modes[i] == MODE_KV:
                ks.append(data[i][0][a:b])
                vs.append(data[i][1][a:b])
            else:
                xs.append(data[i][a:b])
        pool.append(ids, list(w.modes), toks, torch.cat(ks).contiguous(), torch.cat(vs).contiguous(),
                    torch.cat(xs).contiguous())
        o, l = pool.decode(ids, q, w.scale)
        outs[p].copy_(o)
        lses[p].copy_(l)
    out = torch.empty((len(n), d), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((len(n), Hh), dtype=torch.float32, device=dev)
    H.hc_merge_partials(outs[:P], lses[:P], out, lse)
    torch.cuda.synchronize()
    err, lerr = T.compare(w, out.float().cpu().numpy(), lse.cpu().numpy(), range(len(n)))
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE, lerr
    outs[P].fill_(float("nan"))
    lses[P].fill_(float("-inf"))
    out2, lse2 = torch.empty_like(out), torch.empty_like(lse)
    H.hc_merge_partials(outs, lses, out2, lse2)
    torch.cuda.synchronize()
    assert torch.equal(out2, out) and torch.equal(lse2, lse)


# ------------------------------------------------------------------ attention layer (NEXT row f1)
LAYER_CASES = [
    ("tiny-f32", None),
    ("bf16-256", (256, 2, 128, 16)),     # 3d = 768: 256-wide pair tiles for the projection GEMM
    ("bf16-512", (512, 4, 128, 16)),     # 3d = 1536: 512-wide pair tiles
    ("bf16-dh64", (512, 8, 64, 32)),
]


@pytest.mark.parametrize("name,shape", LAYER_CASES)
def test_decode_layer_vs_oracle(hc, name, shape):
    """x_t -> [q,k,v = W x_t, k/v or x_t appended] -> attention -> y = W_O o (+b), against
    oracle.attention_layer; the appended K/V (or x_t) are then re-checked by a plain
    decode_attention over the updated cache."""
    if shape is None:
        w = C.tiny(bias=True)
        tol = TOL_F32
    else:
        d, H, dh, B = shape
        w = _bf16_workload(d, H, dh, B, n=[1, 2, 17, 129, 300, 33], bias=True)
        tol = TOL_BF16
    dev = torch.device("cuda", 0)
    pool = T.make_layer_pool(w)
    T.fill(pool, T.prefix_workload(w))
    x = torch.stack([w.x_t(i, device=dev) for i in range(len(w.n))]).contiguous()
    y, lse = pool.decode_layer(w.req_ids, w.modes, x, w.scale)
    torch.cuda.synchronize()
    y, lse = y.float().cpu().numpy(), lse.cpu().numpy()
    from oracle import hc_oracle as O
    for i in range(len(w.n)):
        y_ref, q_ref, l_ref, ctx = T.oracle_layer(w, i)
        assert O.max_rel_err(y[i][None], y_ref[None], w.shape.H) <= tol, (name, i)
        assert np.abs(lse[i] - l_ref).max() <= (1e-4 if shape is None else TOL_LSE), (name, i)
        assert pool.request_info(w.req_ids[i])[1] == w.n[i]
    # the cache now holds the current token: attend again with the layer's own q
    q = torch.stack([torch.tensor(T.oracle_layer(w, i)[1]) for i in range(len(w.n))]).to(w.torch_dtype).to(dev)
    out, lse2 = pool.decode(w.req_ids, q.contiguous(), w.scale)
    out = out.float().cpu().numpy()
    for i in range(len(w.n)):
        _, q_ref, _, ctx = T.oracle_layer(w, i)
        qd = q.float().cpu().numpy()[i]
        if ctx["mode"] == 1:
            K, V = O.hidden_request_kv(ctx["X"], w.w_kv(), w.b_kv())
        else:
            K, V = ctx["K"], ctx["V"]
        ref, _ = O.attend(qd, K, V, w.shape.H, w.scale)
        assert O.max_rel_err(out[i][None], ref[None], w.shape.H) <= tol, (name, "cache", i)


def test_project_append_errors(hc):
    w = _bf16_workload(256, 2, 128, 16, n=[5])
    pool = T.make_pool(w)       # created without w_q / w_o
    x = torch.zeros((1, 256), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(hc.HcError) as e:
        pool.project_append([0], [0], x)
    assert e.value.status == hc.HC_E_UNSUPPORTED
    with pytest.raises(hc.HcError) as e:
        pool.output_projection(x)
    assert e.value.status == hc.HC_E_UNSUPPORTED


# ------------------------------------------------------------------ prefill / recompute (NEXT row f3)
PREFILL_CASES = [
    ("tiny-f32", None, [64, 1, 33, 16]),
    ("bf16-256", (256, 2, 128, 16), [1, 63, 64, 65, 200, 513]),
    ("bf16-512", (512, 4, 128, 16), [130, 7, 64, 300]),
    ("bf16-dh64", (512, 8, 64, 32), [1, 65, 129]),
    ("bf16-long", (512, 4, 128, 16), [1, 127, 128, 129, 700, 1500]),     # many 128-query tiles
    ("bf16-dh64-long", (512, 8, 64, 32), [255, 256, 257, 1031]),
]


@pytest.mark.parametrize("prefill_tc", ["1", "0"])
@pytest.mark.parametrize("name,shape,lens", PREFILL_CASES)
def test_prefill_layer_vs_oracle(hc, monkeypatch, name, shape, lens, prefill_tc):
    """Prefill of new requests: every output row against oracle.prefill_layer, then a decode
    over the freshly written caches against the oracle (KV rows written by the projection
    GEMM's epilogue; hidden rows = x).  prefill_tc: the tcgen05 attention kernel (default)
    and the mma.sync one (HC_PREFILL_TC=0) meet the same bar."""
    from oracle import hc_oracle as O
    monkeypatch.setenv("HC_PREFILL_TC", prefill_tc)
    if shape is None:
        w = C.tiny(bias=True)
        tol = TOL_F32
    else:
        d, H, dh, B = shape
        w = _bf16_workload(d, H, dh, B, n=lens, bias=True)
        tol = TOL_BF16
    dev = torch.device("cuda", 0)
    pool = T.make_layer_pool(w)
    x = torch.cat([w.x(i, device=dev) for i in range(len(w.n))]).contiguous()
    y = pool.prefill_layer(w.req_ids, w.modes, w.n, x, w.scale)
    torch.cuda.synchronize()
    y = y.float().cpu().numpy()
    W_q, W_kv, W_o = w.w_q(), w.w_kv(), w.w_o()
    r = 0
    for i in range(len(w.n)):
        Y, K, V = O.prefill_layer(w.x(i), W_q, W_kv, W_o, w.shape.H, w.scale, w.b_q(), w.b_kv(), w.b_o())
        assert O.max_rel_err(y[r:r + w.n[i]], Y, w.shape.H) <= tol, (name, i)
        r += w.n[i]
    # the caches now hold every token: decode with the synthetic queries
    out, lse = T.decode(pool, w, T.queries(w))
    for i in range(len(w.n)):
        K, V = O.hidden_request_kv(w.x(i), W_kv, w.b_kv())
        ref, _ = O.attend(w.q(i).double().numpy(), K, V, w.shape.H, w.scale)
        assert O.max_rel_err(out[i][None], ref[None], w.shape.H) <= tol, (name, "cache", i)


def test_recompute_after_cache_type_switch(hc):
    """a request switching KV -> hidden discards its cache and is recomputed by a
    prefill over its tokens in the new mode; decode then matches the oracle."""
    from oracle import hc_oracle as O
    w = _bf16_workload(256, 2, 128, 16, n=[77], modes=[MODE_KV], bias=True)
    dev = torch.device("cuda", 0)
    pool = T.make_layer_pool(w, num_blocks=32)
    x = w.x(0, device=dev)
    pool.prefill_layer(w.req_ids, [MODE_KV], w.n, x, w.scale)
    with pytest.raises(hc.HcError):
        pool.prefill_layer(w.req_ids, [MODE_KV], w.n, x, w.scale)   # not a new request
    assert pool.free(w.req_ids[0]) == 2 * math.ceil(77 / 16)
    pool.prefill_layer(w.req_ids, [MODE_HIDDEN], w.n, x, w.scale)
    assert pool.request_info(w.req_ids[0])[:2] == (MODE_HIDDEN, 77)
    out, _ = pool.decode(w.req_ids, T.queries(w), w.scale)
    K, V = O.hidden_request_kv(w.x(0), w.w_kv(), w.b_kv())
    ref, _ = O.attend(w.q(0).double().numpy(), K, V, 2, w.scale)
    assert O.max_rel_err(out.float().cpu().numpy(), ref[None], 2) <= TOL_BF16


# ------------------------------------------------------------------ RoPE (NEXT row f4)
ROPE_THETA = 500000.0   # LLaMA-3 base


@pytest.mark.parametrize("shape", [(512, 4, 128, 16), (512, 8, 64, 32)])
def test_rope_decode_vs_oracle(hc, monkeypatch, shape):
    """Rebuilt K rows rotated at their token positions in the GEMM epilogue (fused and
    two-kernel paths), contexts up to 3000 tokens."""
    d, H, dh, B = shape
    w = _bf16_workload(d, H, dh, B, n=[1, 17, 300, 3000, 129, 64], bias=True)
    for fused in ("1", "0"):
        monkeypatch.setenv("HC_FUSED", fused)
        pool = T.make_pool(w, rope_theta=ROPE_THETA)
        T.fill(pool, w)
        out, lse = T.decode(pool, w, T.queries(w))
        err, lerr = T.compare(w, out, lse, range(len(w.n)), rope_theta=ROPE_THETA)
        assert err <= TOL_BF16, (fused, err)
        pool.close()


def test_rope_layer_and_prefill_vs_oracle(hc):
    """q and k rotated at the new tokens' positions by the projection epilogue (decode
    layer) and at 0..L-1 (prefill)."""
    from oracle import hc_oracle as O
    d, H, dh, B = 512, 4, 128, 16
    dev = torch.device("cuda", 0)
    w = _bf16_workload(d, H, dh, B, n=[1, 40, 700, 129], bias=True)
    pool = T.make_layer_pool(w, rope_theta=ROPE_THETA)
    T.fill(pool, T.prefix_workload(w))
    x = torch.stack([w.x_t(i, device=dev) for i in range(len(w.n))]).contiguous()
    y, lse = pool.decode_layer(w.req_ids, w.modes, x, w.scale)
    y = y.float().cpu().numpy()
    for i in range(len(w.n)):
        y_ref, _, _, _ = T.oracle_layer(w, i, rope_theta=ROPE_THETA)
        assert O.max_rel_err(y[i][None], y_ref[None], H) <= TOL_BF16, ("layer", i)
    w2 = _bf16_workload(d, H, dh, B, n=[65, 1, 300], bias=True, seed=13)
    pool2 = T.make_layer_pool(w2, rope_theta=ROPE_THETA)
    xs = torch.cat([w2.x(i, device=dev) for i in range(len(w2.n))]).contiguous()
    yp = pool2.prefill_layer(w2.req_ids, w2.modes, w2.n, xs, w2.scale).float().cpu().numpy()
    r = 0
    for i in range(len(w2.n)):
        Y, _, _ = O.prefill_layer(w2.x(i), w2.w_q(), w2.w_kv(), w2.w_o(), H, w2.scale, w2.b_q(), w2.b_kv(),
                                  w2.b_o(), ROPE_THETA)
        assert O.max_rel_err(yp[r:r + w2.n[i]], Y, H) <= TOL_BF16, ("prefill", i)
        r += w2.n[i]


def test_rope_unsupported_paths(hc):
    with pytest.raises(hc.HcError) as e:
        T.make_pool(C.tiny(), rope_theta=10000.0)      # fp32 / SIMT path
    assert e.value.status == hc.HC_E_UNSUPPORTED


# ------------------------------------------------------------------ absorbed hidden attention (NEXT row f4 (ii))
ABSORB_SHAPES = [
    (256, 2, 128, 16),
    (512, 8, 64, 32),
    (384, 3, 128, 8),
    (256, 2, 128, 256),
    (1152, 9, 128, 16),     # H = 9: score/Z tiles padded to 16 heads
    (4608, 72, 64, 16),     # OPT-66B head count (Hp = 80: two 64-column halves of P)
]


@pytest.mark.parametrize("d,H,dh,B", ABSORB_SHAPES)
def test_absorbed_mixed_batch_vs_oracle(hc, d, H, dh, B):
    """HC_FLAG_ABSORB_HIDDEN: hidden requests through q~ = W_K^T q and W_V (sum a x), KV
    requests through split-K attention; same oracle (Eq. 1-3), same bf16 bar."""
    w = _bf16_workload(d, H, dh, B, bias=True)
    pool, out, lse = _run(w, flags=hc.HC_FLAG_ABSORB_HIDDEN)
    assert pool.last_decode_path() == 3
    assert pool.last_launch_count() == 7      # q~, scores, rescale, Z, W_V, attention, combine
    err, lerr = T.compare(w, out, lse, range(len(w.n)))
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE, lerr


def test_absorbed_hidden_only_and_kv_only(hc):
    n = [700, 1, 333, 1025, 64, 65, 4000]
    w = _bf16_workload(512, 4, 128, 16, n=n, modes=[MODE_HIDDEN] * len(n), bias=True)
    pool, out, lse = _run(w, flags=hc.HC_FLAG_ABSORB_HIDDEN)
    assert pool.last_launch_count() == 6      # no KV request: no attention kernel
    assert T.compare(w, out, lse, range(len(n)))[0] <= TOL_BF16
    w = _bf16_workload(512, 4, 128, 16, n=n, modes=[MODE_KV] * len(n), bias=True)
    pool, out, lse = _run(w, flags=hc.HC_FLAG_ABSORB_HIDDEN)
    assert pool.last_decode_path() == 2
    assert T.compare(w, out, lse, range(len(n)))[0] <= TOL_BF16


def test_absorbed_matches_reconstruction_path(hc):
    """Both hidden-mode paths approximate the same fp64 result; they agree with each other
    within twice the bar and the KV rows are bit-identical (same kernels)."""
    w = _bf16_workload(512, 4, 128, 16, bias=True)
    _, a, la = _run(w, split_tokens=64)
    _, b, lb = _run(w, flags=hc.HC_FLAG_ABSORB_HIDDEN, split_tokens=64)
    kv = [i for i in range(len(w.n)) if w.modes[i] == MODE_KV]
    assert np.array_equal(a[kv], b[kv]) and np.array_equal(la[kv], lb[kv])
    from oracle import hc_oracle as O
    assert O.max_rel_err(a, b, 4) <= 2 * TOL_BF16


def test_absorbed_opt66b_sampled(hc):
    """cfg4 (OPT-66B, 256 requests, 50% hidden) in the bench's absorbed configuration."""
    w = C.by_name("cfg4")
    pool = T.make_pool(w, flags=hc.HC_FLAG_ABSORB_HIDDEN)
    T.fill(pool, w)
    out, lse = T.decode(pool, w, T.queries(w))
    assert np.isfinite(out).all()
    idx = _sample(w)
    heads = {i: [0, w.shape.H // 2, w.shape.H - 1] for i in idx if w.modes[i] == MODE_HIDDEN}
    err, lerr = T.compare(w, out[idx], lse[idx], idx, heads)
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE, lerr


def test_absorbed_decode_layer(hc):
    """hc_decode_layer on an absorbed pool: projection, append, absorbed attention, W_O."""
    from oracle import hc_oracle as O
    d, H, dh, B = 512, 4, 128, 16
    dev = torch.device("cuda", 0)
    w = _bf16_workload(d, H, dh, B, n=[1, 40, 700, 129, 2, 3000], bias=True)
    pool = T.make_layer_pool(w, flags=hc.HC_FLAG_ABSORB_HIDDEN)
    T.fill(pool, T.prefix_workload(w))
    x = torch.stack([w.x_t(i, device=dev) for i in range(len(w.n))]).contiguous()
    y, lse = pool.decode_layer(w.req_ids, w.modes, x, w.scale)
    y = y.float().cpu().numpy()
    for i in range(len(w.n)):
        y_ref, _, _, _ = T.oracle_layer(w, i)
        assert O.max_rel_err(y[i][None], y_ref[None], H) <= TOL_BF16, i


def test_absorbed_unsupported_configs(hc):
    for kw in ({"rope_theta": 10000.0}, {}):
        w = C.tiny() if not kw else _bf16_workload(512, 4, 128, 16)
        with pytest.raises(hc.HcError) as e:
            T.make_pool(w, flags=hc.HC_FLAG_ABSORB_HIDDEN, **kw)   # RoPE / fp32
        assert e.value.status == hc.HC_E_UNSUPPORTED



# ------------------------------------------------------------------ pre-attention LayerNorm (f1 option, R15)
LN_CASES = [("tiny-f32", None), ("bf16-512", (512, 4, 128, 16)), ("bf16-dh64", (512, 8, 64, 32))]
# A layer with LayerNorm stores u = LN(x) in the pool dtype before q, k, v (the hidden cache
# holds it, R15); the oracle takes that stored vector, u = bf16(LN(x)) (reading R16), so the
# bf16 bar stays north_star's 1e-2.  fp32 keeps 1e-5.


def _ln_input(t):
    """Layer inputs with a non-zero mean and a non-unit scale (so LN matters), made on the
    host and copied to the device (the oracle reads the host copy)."""
    return (t.float() * 2.5 + 1.0).to(t.dtype)


@pytest.mark.parametrize("name,shape", LN_CASES)
def test_layer_norm_and_decode_layer_with_ln(hc, name, shape):
    from oracle import hc_oracle as O
    if shape is None:
        w, tol = C.tiny(bias=True), TOL_F32
    else:
        w, tol = _bf16_workload(*shape, n=[1, 40, 700, 129, 2], bias=True), TOL_BF16
    dev = torch.device("cuda", 0)
    pool = T.make_layer_pool(w, ln=True)
    ln = T.ln_params(w, store=w.dtype)
    xs = [_ln_input(w.x_t(i)) for i in range(len(w.n))]
    x = torch.stack(xs).contiguous().to(dev)
    # hc_layer_norm alone: every element within the storage precision of the fp64 LN
    u = pool.layer_norm(x).float().cpu().numpy()
    ref = O.layer_norm(torch.stack(xs), *ln[:3])
    assert np.abs(u - ref).max() <= (1e-5 if shape is None else 2e-2) * max(1.0, np.abs(ref).max())
    T.fill(pool, T.prefix_workload(w))
    y, lse = pool.decode_layer(w.req_ids, w.modes, x, w.scale)
    y = y.float().cpu().numpy()
    for i in range(len(w.n)):
        y_ref, _, _, _ = T.oracle_layer(w, i, ln=ln, x_t=xs[i])
        assert O.max_rel_err(y[i][None], y_ref[None], w.shape.H) <= tol, (name, i)


@pytest.mark.parametrize("name,shape", LN_CASES)
def test_prefill_with_ln_then_decode(hc, name, shape):
    """Prefill with LN: outputs against the oracle, then a decode over the written caches —
    hidden caches hold u = LN(x), KV caches hold W_KV u (+b)."""
    from oracle import hc_oracle as O
    if shape is None:
        w, tol = C.tiny(bias=True), TOL_F32
    else:
        w, tol = _bf16_workload(*shape, n=[65, 1, 300, 129], bias=True, seed=17), TOL_BF16
    dev = torch.device("cuda", 0)
    pool = T.make_layer_pool(w, ln=True)
    ln = T.ln_params(w, store=w.dtype)
    X = [_ln_input(w.x(i)) for i in range(len(w.n))]
    yp = pool.prefill_layer(w.req_ids, w.modes, w.n, torch.cat(X).contiguous().to(dev), w.scale)
    yp = yp.float().cpu().numpy()
    r = 0
    for i in range(len(w.n)):
        Y, _, _ = O.prefill_layer(X[i], w.w_q(), w.w_kv(), w.w_o(), w.shape.H, w.scale, w.b_q(), w.b_kv(),
                                  w.b_o(), ln=ln)
        assert O.max_rel_err(yp[r:r + w.n[i]], Y, w.shape.H) <= tol, (name, "prefill", i)
        r += w.n[i]
    out, _ = T.decode(pool, w, T.queries(w))
    for i in range(len(w.n)):
        K, V = O.hidden_request_kv(O.layer_norm(X[i], *ln), w.w_kv(), w.b_kv())
        ref, _ = O.attend(w.q(i).double().numpy(), K, V, w.shape.H, w.scale)
        assert O.max_rel_err(out[i][None], ref[None], w.shape.H) <= tol, (name, "cache", i)


def test_layer_norm_unconfigured_is_unsupported(hc):
    w = _bf16_workload(512, 4, 128, 16, n=[3])
    pool = T.make_layer_pool(w)
    with pytest.raises(hc.HcError) as e:
        pool.layer_norm(torch.zeros(2, 512, dtype=torch.bfloat16, device="cuda"))
    assert e.value.status == hc.HC_E_UNSUPPORTED


# ------------------------------------------------------------------ fused reconstruct-and-attend (f1)
@pytest.mark.parametrize("shape", [(512, 4, 128, 16), (512, 8, 64, 32), (384, 3, 128, 8), (256, 2, 128, 256),
                                   (256, 8, 32, 16)])
def test_attend_epilogue_vs_scratch_path(hc, monkeypatch, shape):
    """The default bf16 path turns rebuilt K/V into flash-decoding partials inside the GEMM
    epilogue (segments of min(B, 32) tokens; K/V never stored).  It meets the oracle bar,
    agrees with the K/V-scratch path (HC_EPI_ATTEND=0) within twice the bar with bit-identical
    KV-mode rows, and needs far less workspace."""
    d, H, dh, B = shape
    w = _bf16_workload(d, H, dh, B, bias=True)
    pool, a, la = _run(w, split_tokens=64)
    ids = list(w.req_ids)
    ws_attend = pool.workspace_size(ids)
    assert T.compare(w, a, la, range(len(w.n)))[0] <= TOL_BF16
    monkeypatch.setenv("HC_EPI_ATTEND", "0")
    pool2, b, lb = _run(w, split_tokens=64)
    from oracle import hc_oracle as O
    assert O.max_rel_err(a, b, H) <= 2 * TOL_BF16
    kv = [i for i in range(len(w.n)) if w.modes[i] == MODE_KV]
    assert np.array_equal(a[kv], b[kv]) and np.array_equal(la[kv], lb[kv])
    assert ws_attend < pool2.workspace_size(ids)


def test_attend_epilogue_rope_and_long_contexts(hc):
    """RoPE applied to k in registers before the dot product; contexts spanning many
    segments and a last segment past n inside the last block."""
    w = _bf16_workload(512, 4, 128, 16, n=[1, 17, 300, 4000, 129, 64, 2049], bias=True)
    pool = T.make_pool(w, rope_theta=ROPE_THETA)
    T.fill(pool, w)
    out, lse = T.decode(pool, w, T.queries(w))
    err, lerr = T.compare(w, out, lse, range(len(w.n)), rope_theta=ROPE_THETA)
    assert err <= TOL_BF16 and lerr <= TOL_LSE, (err, lerr)


# ------------------------------------------------------------------ where the kernels are most fragile
def _opt66_workload(n, modes, seed, q_scale=1.0, bias=True):
    shape = LayerShape("opt66b-shape", 9216, 72, 128)
    return Workload(f"frag-{seed}", shape, 16, "bf16", seed, list(n), list(modes), list(range(len(n))), bias,
                    q_scale=q_scale)


@pytest.mark.parametrize("q_scale", [4.0, 32.0])
def test_high_dynamic_range_softmax_on_the_fused_path(hc, q_scale):
    """Eq. 2 with peaky scores: q x4 (SURVEY §8(d) "peaky" variant, scores ~N(0, 16)) and q x32
    (scores ~N(0, 1024): softmax is an argmax, out -> v_argmax; exercises the online rescale and
    the exp2 path in both the KV warps and the attend epilogue).  OPT-66B head shape, all heads."""
    n = [1, 17, 600, 300, 33, 129, 2, 257]
    modes = [MODE_HIDDEN, MODE_KV, MODE_KV, MODE_HIDDEN, MODE_HIDDEN, MODE_KV, MODE_KV, MODE_HIDDEN]
    w = _opt66_workload(n, modes, seed=41 + int(q_scale), q_scale=q_scale)
    pool, out, lse = _run(w)
    assert pool.last_decode_path() == 1
    assert np.isfinite(out).all() and np.isfinite(lse).all()
    err, lerr = T.compare(w, out, lse, range(len(n)))
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE * max(1.0, float(np.abs(lse).max()) / 10), lerr


@pytest.mark.parametrize("cfg", ["cfg4", "cfg5:1/32"])
def test_all_heads_of_the_longest_hidden_request_full_size(hc, cfg):
    """Full-size batch in the bench's launch configuration; the oracle checks EVERY head of the
    longest hidden request (all 36 GEMM n-tiles at d = 9216), of 3 more hidden requests and of
    24 KV-mode requests including the longest."""
    w = C.by_name(cfg)
    pool = T.make_pool(w)
    T.fill(pool, w)
    out, lse = T.decode(pool, w, T.queries(w))
    hid = [i for i in range(len(w.n)) if w.modes[i] == MODE_HIDDEN]
    kv = [i for i in range(len(w.n)) if w.modes[i] == MODE_KV]
    rs = np.random.default_rng(5)
    longest = max(hid, key=lambda i: w.n[i])
    others = [i for i in hid if i != longest]
    kv_longest = max(kv, key=lambda i: w.n[i])
    kv_pick = [kv_longest] + [int(i) for i in rs.choice([i for i in kv if i != kv_longest], size=23, replace=False)]
    idx = [longest] + [int(i) for i in rs.choice(others, size=min(3, len(others)), replace=False)] + kv_pick
    err, lerr = T.compare(w, out[idx], lse[idx], idx)
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE, lerr


def test_split_and_segment_boundary_lengths_at_d9216(hc):
    """Context lengths on either side of every boundary the kernels have: the 16-token KV
    chunk and block, the 32-token attend segment, the 512-token auto split (and 2x, 3x), for
    both cache modes, in one fused batch at OPT-66B shape.  KV requests: all heads; hidden
    requests: heads 0, 35, 71 (first, middle and last GEMM n-tiles)."""
    lens = [15, 16, 17, 31, 32, 33, 511, 512, 513, 1023, 1024, 1025, 1535, 1536, 1537]
    n = lens + lens
    modes = [MODE_KV] * len(lens) + [MODE_HIDDEN] * len(lens)
    w = _opt66_workload(n, modes, seed=77)
    pool, out, lse = _run(w)
    assert pool.last_decode_path() == 1
    heads = {i: [0, 35, 71] for i in range(len(n)) if modes[i] == MODE_HIDDEN}
    err, lerr = T.compare(w, out, lse, range(len(n)), heads)
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE, lerr


def test_failed_append_after_allocation_leaves_the_pool_unchanged(hc):
    """hc.h: errors leave the pool unchanged.  With all 16 pinned staging slots held by captured
    CUDA graphs, hc_append fails AFTER allocating (HC_E_CUDA): the request's length, block
    table and the free count must be rolled back, and a retry after the graphs are gone
    appends exactly once."""
    w = _bf16_workload(512, 4, 128, 16, n=[40, 20], modes=[MODE_KV, MODE_HIDDEN])
    pool = T.make_pool(w, num_blocks=64)
    T.fill(pool, w)
    q = T.queries(w)
    ids = list(w.req_ids)
    out = torch.empty_like(q)
    ws = pool.workspace(ids)
    graphs = []
    torch.cuda.synchronize()
    for _ in range(16):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            hc.hc_decode_attention(pool.handle, ids, q, w.scale, out, None, ws, torch.cuda.current_stream())
        graphs.append(g)
    before = (pool.request_info(ids[0]), pool.request_blocks(ids[0], 0), pool.num_free())
    k = torch.zeros((9, 512), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(hc.HcError) as e:
        pool.append([ids[0], 99], [MODE_KV, MODE_KV], [9, 9], k=torch.cat([k, k]), v=torch.cat([k, k]))
    assert e.value.status == hc.HC_E_CUDA
    assert (pool.request_info(ids[0]), pool.request_blocks(ids[0], 0), pool.num_free()) == before
    with pytest.raises(hc.HcError):
        pool.request_info(99)   # the request the failed call would have created does not exist


def test_bench_token_range_split_matches_the_oracle(hc, tmp_path):
    """bench.py --strong --split with 2 ranks (both on this GPU, gloo): a request longer than
    total/world is split into block-aligned token ranges on both ranks, decoded, all-gathered
    and merged by hc_merge_partials; the merged (out, lse) of every request (dumped by the
    bench's HC_BENCH_DUMP hook) equals the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dump = str(tmp_path / "split.npz")
    env = dict(os.environ, HC_BENCH_ONE_GPU="1", HC_BENCH_BACKEND="gloo", HC_BENCH_DUMP=dump)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", "tiny",
                        "--strong", "--split", "--steps", "3", "--warmup", "3"], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = np.load(dump)
    w = C.tiny()
    assert d["parts"].max() >= 2   # at least one request really was split
    err, lerr = T.compare(w, d["out"], d["lse"], range(len(w.n)))
    assert err <= TOL_F32 and lerr <= 1e-5, (err, lerr)


# ------------------------------------------------------------------ grouped-query attention (f4 (i), R18)
GQA_SHAPES = [
    # (d, H, dh, B, Hk): fused tcgen05 path needs dh = 128 and 2*Hk*dh % 512 == 0
    (1024, 8, 128, 16, 2),     # G = 4, Bkv = 32: fused
    (4096, 32, 128, 16, 8),    # LLaMA-3-8B layer: fused
    (4096, 32, 128, 16, 4),    # Yi-6B layer: G = 8, Bkv = 64
    (512, 8, 64, 32, 2),       # dh 64: two-kernel tcgen05 path, Bkv = 64
    (512, 8, 64, 16, 8),       # Hk = H spelled out: multi-head
]


@pytest.mark.parametrize("d,H,dh,B,Hk", GQA_SHAPES)
def test_gqa_decode_vs_oracle(hc, d, H, dh, B, Hk):
    """Mixed KV/hidden batch under GQA: KV tokens take one unit per Bkv = B d / (2 Hk dh) tokens
    (K and V of Bkv tokens in one unit), hidden tokens one unit per B; query head h reads K/V
    head h / G in the KV warps and in the attend epilogue (G query heads per rebuilt K/V head)."""
    n = [1, 17, 300, 129, 64, 511, 33, 1000]
    w = _bf16_workload(d, H, dh, B, n=n, bias=True, Hk=Hk)
    pool, out, lse = _run(w)
    err, lerr = T.compare(w, out, lse, range(len(n)))
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE, lerr
    Bkv = B * d // (2 * Hk * dh) if Hk != H else B
    for i in range(len(n)):
        units = pool.request_info(w.req_ids[i])[2]
        want = -(-n[i] // B) if w.modes[i] == MODE_HIDDEN else (-(-n[i] // Bkv) * (1 if Hk != H else 2))
        assert units == want, (i, units, want)


@pytest.mark.parametrize("env", [{"HC_FUSED": "0"}, {"HC_EPI_ATTEND": "0"}, {"HC_EPI_ATTEND": "0", "HC_FUSED": "0"},
                                 {"HC_ATTN_TC": "0"}, {"HC_ATTN_TC": "0", "HC_FUSED": "0"},
                                 {"HC_GQA_SCRATCH": "1"}, {"HC_GQA_SCRATCH": "1", "HC_FUSED": "0"}])
def test_gqa_alternative_paths(hc, monkeypatch, env):
    """GQA through the two-kernel path, the fused kernel with K/V scratch ([hblock][Hk][B][dh]),
    and the stand-alone GEMM + attention kernel, at the LLaMA-3-8B head layout."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = _bf16_workload(1024, 8, 128, 16, n=[1, 17, 300, 129, 64, 511], bias=True, Hk=2)
    _, out, lse = _run(w, split_tokens=64)
    err, lerr = T.compare(w, out, lse, range(len(w.n)))
    assert err <= TOL_BF16 and lerr <= TOL_LSE, (err, lerr)


def test_gqa_fp32_simt_and_rope(hc):
    """fp32 (SIMT reconstruction + generic attention) under GQA at 1e-5, and bf16 GQA with RoPE
    (rebuilt K rotated per K/V head in the attend epilogue)."""
    sh = LayerShape("gqa-f32", 128, 8, 16, 2)
    w = Workload("gqa-f32", sh, 4, "f32", 5, [9, 1, 6, 40, 13], [MODE_KV, MODE_HIDDEN, MODE_HIDDEN, MODE_KV, MODE_HIDDEN],
                 [0, 1, 2, 3, 4], True)
    _, out, lse = _run(w)
    err, lerr = T.compare(w, out, lse, range(len(w.n)))
    assert err <= TOL_F32 and lerr <= 1e-5, (err, lerr)
    w2 = _bf16_workload(1024, 8, 128, 16, n=[1, 17, 300, 2049, 64], bias=True, Hk=2)
    pool = T.make_pool(w2, rope_theta=ROPE_THETA)
    T.fill(pool, w2)
    out2, lse2 = T.decode(pool, w2, T.queries(w2))
    err2, lerr2 = T.compare(w2, out2, lse2, range(len(w2.n)), rope_theta=ROPE_THETA)
    assert err2 <= TOL_BF16 and lerr2 <= TOL_LSE, (err2, lerr2)


@pytest.mark.parametrize("shape", [(1024, 8, 128, 16, 2), (512, 8, 64, 32, 2)])
def test_gqa_decode_layer_and_prefill_vs_oracle(hc, shape):
    """f1/f3 under GQA: the projection GEMM's epilogue writes q and the K/V rows of the Hk heads
    into the packed KV units; prefill attends with query head h on K/V head h / G."""
    from oracle import hc_oracle as O
    d, H, dh, B, Hk = shape
    w = _bf16_workload(d, H, dh, B, n=[1, 2, 17, 129, 300, 33], bias=True, Hk=Hk)
    dev = torch.device("cuda", 0)
    pool = T.make_layer_pool(w)
    T.fill(pool, T.prefix_workload(w))
    x = torch.stack([w.x_t(i, device=dev) for i in range(len(w.n))]).contiguous()
    y, lse = pool.decode_layer(w.req_ids, w.modes, x, w.scale)
    y = y.float().cpu().numpy()
    for i in range(len(w.n)):
        y_ref, _, _, _ = T.oracle_layer(w, i)
        assert O.max_rel_err(y[i][None], y_ref[None], H) <= TOL_BF16, i
    w2 = _bf16_workload(d, H, dh, B, n=[65, 1, 300, 129], bias=True, seed=19, Hk=Hk)
    pool2 = T.make_layer_pool(w2)
    xp = torch.cat([w2.x(i, device=dev) for i in range(len(w2.n))]).contiguous()
    yp = pool2.prefill_layer(w2.req_ids, w2.modes, w2.n, xp, w2.scale).float().cpu().numpy()
    r = 0
    kv_ref = []
    for i in range(len(w2.n)):
        Y, K, V = O.prefill_layer(w2.x(i), w2.w_q(), w2.w_kv(), w2.w_o(), H, w2.scale, w2.b_q(), w2.b_kv(), w2.b_o())
        assert O.max_rel_err(yp[r:r + w2.n[i]], Y, H) <= TOL_BF16, ("prefill", i)
        kv_ref.append((K, V))
        r += w2.n[i]
    # a decode over the caches prefill wrote (packed KV units hold W_KV x + b; hidden units hold x)
    out, _ = T.decode(pool2, w2, T.queries(w2))
    for i in range(len(w2.n)):
        ref, _ = O.attend(w2.q(i).double().numpy(), *kv_ref[i], H, w2.scale, n_kv_heads=Hk)
        assert O.max_rel_err(out[i][None], ref[None], H) <= TOL_BF16, ("cache", i)


@pytest.mark.parametrize("cfg", ["llama3-8b", "yi-6b"])
def test_gqa_full_size_sampled(hc, cfg):
    """The bench's GQA workloads (LLaMA-3-8B: G = 4, attend epilogue; Yi-6B: G = 8, rebuilt K/V
    scratch + tensor-core loop; 256 requests, long contexts, 50% hidden) in the bench's launch
    configuration; every head of the longest hidden and longest KV request."""
    w = C.by_name(cfg)
    pool = T.make_pool(w)
    T.fill(pool, w)
    out, lse = T.decode(pool, w, T.queries(w))
    assert pool.last_decode_path() == 1 and np.isfinite(out).all()
    hid = [i for i in range(len(w.n)) if w.modes[i] == MODE_HIDDEN]
    kv = [i for i in range(len(w.n)) if w.modes[i] == MODE_KV]
    idx = [max(hid, key=lambda i: w.n[i]), max(kv, key=lambda i: w.n[i]), hid[0], kv[0]]
    err, lerr = T.compare(w, out[idx], lse[idx], idx)
    print(cfg, "max normwise err", err, "lse err", lerr)
    assert err <= TOL_BF16 and lerr <= TOL_LSE, (err, lerr)


def test_gqa_refused_with_the_absorbed_variant(hc):
    w = _bf16_workload(1024, 8, 128, 16, n=[3], Hk=2)
    with pytest.raises(hc.HcError) as e:
        T.make_pool(w, flags=hc.HC_FLAG_ABSORB_HIDDEN)
    assert e.value.status == hc.HC_E_UNSUPPORTED


@pytest.mark.parametrize("shape", [(512, 4, 128, 16), (512, 8, 64, 32), (9216, 72, 128, 16)])
def test_tensor_core_kv_loop_on_multihead(hc, monkeypatch, shape):
    """HC_ATTN_TC=2: the mma.sync KV loop (attn_tc.cuh) also for multi-head pools — fused
    (attend epilogue + KV warps), KV-only batches (stand-alone kernel) and peaky scores; it
    meets the same bar as the FHFMA SIMT loop."""
    monkeypatch.setenv("HC_ATTN_TC", "2")
    d, H, dh, B = shape
    n = [1, 17, 300, 129, 64, 511, 2049]
    w = _bf16_workload(d, H, dh, B, n=n, bias=True)
    _, out, lse = _run(w)
    err, lerr = T.compare(w, out, lse, range(len(n)), {i: [0, H - 1] for i in range(len(n)) if w.modes[i]} if d > 4096 else None)
    assert err <= TOL_BF16 and lerr <= TOL_LSE, (err, lerr)
    wk = _bf16_workload(d, H, dh, B, n=n, modes=[MODE_KV] * len(n), seed=5)
    w4 = Workload(wk.name, wk.shape, B, "bf16", 5, n, [MODE_KV] * len(n), list(range(len(n))), False, q_scale=4.0)
    _, out, lse = _run(w4)
    err, lerr = T.compare(w4, out, lse, range(len(n)))
    assert err <= TOL_BF16 and lerr <= TOL_LSE, (err, lerr)


# ------------------------------------------------------------------ attend epilogue on mma.sync
EPI_MMA_SHAPES = [
    (4096, 32, 128, 16, 8),    # LLaMA-3-8B layer, G = 4, 16-token segments
    (4096, 32, 128, 16, 4),    # Yi-6B layer, G = 8 (attend path now, not the scratch mode)
    (2048, 16, 128, 32, 4),    # B = 32: 32-token segments (two 16-row groups per segment)
    (1024, 8, 128, 64, 4),     # B = 64: blocks of two segments, G = 2
    (2048, 16, 128, 256, 2),   # B = 256: a block spans a whole M tile, G = 8
]


@pytest.mark.parametrize("q_scale", [1.0, 4.0, 32.0])
@pytest.mark.parametrize("d,H,dh,B,Hk", EPI_MMA_SHAPES)
def test_gqa_mma_epilogue_vs_oracle(hc, d, H, dh, B, Hk, q_scale):
    """The GQA attend epilogue on mma.sync (pair_gemm.cuh attend_tile_mma, default for GQA):
    S = (K_hi + K_lo) Q^T, per-segment softmax, O = P^T V with movmatrix-transposed V fragments.
    Normal, peaky (q x4) and argmax-like (q x32) scores; segment lengths 16 and 32; ragged
    requests (tokens past n inside the last block, rows past M in the last tile)."""
    n = [1, 17, 300, 129, 64, 511, 33, 1000, 16, 15]
    modes = [MODE_HIDDEN if i % 3 != 1 else MODE_KV for i in range(len(n))]
    shape = LayerShape(f"mma-{d}-gqa{Hk}", d, H, dh, Hk)
    w = Workload(f"mma-{d}-{B}", shape, B, "bf16", 23 + int(q_scale), n, modes, list(range(len(n))), True,
                 q_scale=q_scale)
    pool, out, lse = _run(w)
    assert pool.last_decode_path() == 1
    assert np.isfinite(out).all() and np.isfinite(lse).all()
    err, lerr = T.compare(w, out, lse, range(len(n)))
    assert err <= TOL_BF16, err
    assert lerr <= TOL_LSE * max(1.0, float(np.abs(lse).max()) / 10), lerr


def test_gqa_mma_epilogue_agrees_with_the_per_row_epilogue(hc, monkeypatch):
    """HC_EPI_MMA=0 restores the per-row (fp32 CUDA-core) attend epilogue: both within the bf16
    bar of each other, KV-mode rows (same KV warps) bit-identical."""
    d, H, dh, B, Hk = 4096, 32, 128, 16, 8
    w = _bf16_workload(d, H, dh, B, n=[5, 300, 129, 1000, 64], bias=True, Hk=Hk)
    _, a, la = _run(w)
    monkeypatch.setenv("HC_EPI_MMA", "0")
    _, b, lb = _run(w)
    from oracle import hc_oracle as O
    assert O.max_rel_err(a, b, H) <= 2 * TOL_BF16
    kv = [i for i in range(len(w.n)) if w.modes[i] == MODE_KV]
    assert np.array_equal(a[kv], b[kv]) and np.array_equal(la[kv], lb[kv])


@pytest.mark.parametrize("d,H,dh,B,Hk", EPI_MMA_SHAPES)
def test_gqa_mma_epilogue_with_rope(hc, d, H, dh, B, Hk):
    """RoPE inside the mma epilogue: columns c and c + 64 of K are the 16x256b slices kk and
    kk + 4, rotated in registers at each row's token position before the hi/lo split; long
    contexts (positions into the thousands) and ragged last blocks."""
    n = [1, 17, 300, 4000, 129, 64, 2049, 33]
    modes = [MODE_HIDDEN if i % 3 != 1 else MODE_KV for i in range(len(n))]
    shape = LayerShape(f"mma-rope-{d}-gqa{Hk}", d, H, dh, Hk)
    w = Workload(f"mma-rope-{d}-{B}", shape, B, "bf16", 31, n, modes, list(range(len(n))), True)
    pool = T.make_pool(w, rope_theta=ROPE_THETA)
    T.fill(pool, w)
    out, lse = T.decode(pool, w, T.queries(w))
    assert pool.last_decode_path() == 1
    err, lerr = T.compare(w, out, lse, range(len(n)), rope_theta=ROPE_THETA)
    assert err <= TOL_BF16 and lerr <= TOL_LSE, (err, lerr)


@pytest.mark.parametrize("env", [{"HC_DYN_TILES": "0"}, {"HC_FUSED_CFG": "3424"}, {"HC_GROUP_N": "2"}])
def test_gqa_mma_epilogue_schedules_agree_bitwise(hc, monkeypatch, env):
    """GQA through the mma epilogue: the static tile stride vs the dynamic tile queue, another
    fused configuration, another raster — only the order of whole tiles / tasks changes =>
    identical bits."""
    d, H, dh, B, Hk = 2048, 16, 128, 16, 4
    n = [700, 33, 511, 1, 257, 96, 129, 64, 300, 17]
    modes = [MODE_HIDDEN if i % 4 != 1 else MODE_KV for i in range(len(n))]
    w = _bf16_workload(d, H, dh, B, n=n, modes=modes, bias=True, Hk=Hk)
    _, a, la = _run(w, split_tokens=64)
    assert T.compare(w, a, la, range(len(n)))[0] <= TOL_BF16
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, b, lb = _run(w, split_tokens=64)
    assert np.array_equal(a, b) and np.array_equal(la, lb)
