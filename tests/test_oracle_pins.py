"""Pins the fp64 oracle to things other than itself (task rule ③).

Each test names the passage / closed form it pins.  Together they are chosen so that a
plausible mistake in oracle/hc_oracle.py (a dropped bias, a wrong sign in the softmax
shift, a transposed W, a wrong head slice, a wrong scale, v_i instead of v_j) fails at
least one of them.
"""
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest
import torch

from oracle import hc_oracle as O
from synth import configs as C


# ---------------------------------------------------------------- Decimal brute force
def _dec_attend(q, K, V, H, scale):
    """40-digit Decimal Eq. 2-3 written from the paper with plain loops."""
    getcontext().prec = 40
    n, d = len(K), len(q)
    dh = d // H
    sc = Decimal(repr(scale))
    out, lse = [Decimal(0)] * d, []
    for h in range(H):
        cols = range(h * dh, (h + 1) * dh)
        s = [sc * sum(Decimal(repr(float(q[c]))) * K[j][c] for c in cols) for j in range(n)]
        m = max(s)
        e = [(x - m).exp() for x in s]
        z = sum(e)
        for c in cols:
            out[c] = sum(e[j] / z * V[j][c] for j in range(n))
        lse.append(m + z.ln())
    return out, lse


def _dec_matrix(t):
    return [[Decimal(repr(float(v))) for v in row] for row in t.tolist()]


def _dec_recon(X, W, b):
    """k_j = W x_j + b with Decimal sums (Eq. 1)."""
    out = []
    for x in X:
        row = []
        for wr, bb in zip(W, b):
            row.append(sum(wv * xv for wv, xv in zip(wr, x)) + bb)
        out.append(row)
    return out


@pytest.mark.parametrize("bias", [False, True])
def test_oracle_vs_decimal_bruteforce_tiny(bias):
    """tiny config (4 requests, d=32, 2x16 heads; KV and hidden) vs 40-digit Decimal.
    Pins Eq. 1 (orientation of W, bias), Eq. 2 (scale, max shift, normalisation) and
    Eq. 3 (v_j weighting) to 1e-13 relative."""
    w = C.tiny(bias=bias)
    d, H = w.shape.d, w.shape.H
    W = w.w_kv()
    b = w.b_kv()
    Wd = _dec_matrix(W.double())
    bd = [Decimal(repr(float(v))) for v in (b.tolist() if b is not None else [0.0] * (2 * d))]
    for i in range(4):
        q = w.q(i).double().numpy()
        if w.modes[i] == C.MODE_KV:
            K, V = w.kv(i)
            Kd, Vd = _dec_matrix(K.double()), _dec_matrix(V.double())
            req = {"mode": 0, "q": q, "K": K, "V": V}
        else:
            X = w.x(i)
            Xd = _dec_matrix(X.double())
            Kd = _dec_recon(Xd, Wd[:d], bd[:d])
            Vd = _dec_recon(Xd, Wd[d:], bd[d:])
            req = {"mode": 1, "q": q, "X": X}
        out_ref, lse_ref = _dec_attend(q, Kd, Vd, H, w.scale)
        out, lse = O.decode_batch([req], W, H, w.scale, b)
        for c in range(d):
            ref = float(out_ref[c])
            assert abs(out[0, c] - ref) <= 1e-13 * max(1.0, abs(ref))
        for h in range(H):
            assert abs(lse[0, h] - float(lse_ref[h])) <= 1e-13 * max(1.0, abs(float(lse_ref[h])))


# ---------------------------------------------------------------- closed forms
def _rand(shape, seed, scale=1.0):
    return np.random.default_rng(seed).normal(0, scale, size=shape)


def test_identity_weights_reconstruct_exactly():
    """W_K = W_V = I  =>  K = V = X exactly (Eq. 1 with identity maps)."""
    X = _rand((7, 12), 0)
    K, V = O.reconstruct_kv(X, np.eye(12), np.eye(12))
    assert np.array_equal(K, X) and np.array_equal(V, X)


def test_permutation_weights_permute_columns():
    """W = permutation matrix P (k = P x)  =>  k_j[r] = x_j[perm[r]] exactly; catches W vs W^T."""
    perm = np.random.default_rng(1).permutation(10)
    P = np.zeros((10, 10))
    P[np.arange(10), perm] = 1.0
    X = _rand((5, 10), 2)
    K, _ = O.reconstruct_kv(X, P, np.eye(10))
    assert np.array_equal(K, X[:, perm])


def test_single_token_returns_v1():
    """n = 1: a_11 = 1 (Eq. 2), so out = v_1 (north_star invariant); hidden: W_V x_1 + b_V."""
    d, H = 16, 4
    q, K, V = _rand(d, 3), _rand((1, d), 4), _rand((1, d), 5)
    out, lse = O.attend(q, K, V, H, 0.25)
    assert np.allclose(out, V[0], rtol=0, atol=1e-15)
    s = [0.25 * q[h * 4:(h + 1) * 4] @ K[0, h * 4:(h + 1) * 4] for h in range(H)]
    assert np.allclose(lse, s, atol=1e-15)
    X, W, b = _rand((1, d), 6), _rand((2 * d, d), 7), _rand(2 * d, 8)
    out2, _ = O.decode_batch([{"mode": 1, "q": q, "X": X}], W, H, 0.25, b)
    assert np.allclose(out2[0], W[d:] @ X[0] + b[d:], atol=1e-13)


def test_zero_query_gives_mean_of_values():
    """q = 0  =>  all scores equal  =>  a_j = 1/n  =>  out = mean_j v_j."""
    d, n = 8, 9
    out, lse = O.attend(np.zeros(d), _rand((n, d), 9), V := _rand((n, d), 10), 2, 0.5)
    assert np.allclose(out, V.mean(axis=0), atol=1e-14)
    assert np.allclose(lse, math.log(n), atol=1e-14)


def test_constant_values_give_constant_output_and_probs_sum_to_one():
    """V = 1  =>  out = sum_j a_j = 1 (softmax rows sum to 1, north_star invariant)."""
    d, n, H = 16, 33, 2
    out, lse, a = O.attend(_rand(d, 11, 3.0), _rand((n, d), 12), np.ones((n, d)), H, 1.0,
                           return_probs=True)
    assert np.allclose(out, 1.0, atol=1e-14)
    assert np.allclose(a.sum(axis=1), 1.0, atol=1e-14)
    assert (a > 0).all()


def test_key_bias_is_a_per_head_score_shift():
    """b_K adds q_h . b_K,h to every score of head h: output unchanged, lse shifted by
    scale * q_h . b_K,h (catches a dropped / misplaced key bias and the max shift sign)."""
    d, n, H, sc = 16, 20, 2, 0.3
    X, W, q = _rand((n, d), 13), _rand((2 * d, d), 14, 0.25), _rand(d, 15)
    bK = _rand(d, 16)
    b = np.concatenate([bK, np.zeros(d)])
    o0, l0 = O.decode_batch([{"mode": 1, "q": q, "X": X}], W, H, sc)
    o1, l1 = O.decode_batch([{"mode": 1, "q": q, "X": X}], W, H, sc, b)
    assert np.allclose(o0, o1, atol=1e-12)
    shift = [sc * q[h * 8:(h + 1) * 8] @ bK[h * 8:(h + 1) * 8] for h in range(H)]
    assert np.allclose(l1[0] - l0[0], shift, atol=1e-12)


def test_large_scale_selects_argmax_value():
    """scale -> large with a unique maximal score  =>  out -> v_argmax (Eq. 2 limit)."""
    d, n = 8, 6
    q, K, V = _rand(d, 17), _rand((n, d), 18), _rand((n, d), 19)
    j = int(np.argmax(K @ q))
    out, _ = O.attend(q, K, V, 1, 1e4)
    assert np.allclose(out, V[j], atol=1e-9)


def test_matches_torch_sdpa_float64_multihead():
    """Library routine: all-KV batch with H heads == torch SDPA (float64, one query).
    Pins the head slicing (columns h*dh..h*dh+dh-1) and the explicit scale."""
    d, H, n = 48, 3, 17
    q, K, V = _rand(d, 20), _rand((n, d), 21), _rand((n, d), 22)
    sc = 1.0 / math.sqrt(d // H)
    out, _ = O.attend(q, K, V, H, sc)
    tq = torch.tensor(q).view(1, H, 1, d // H)
    tk = torch.tensor(K).view(n, H, d // H).transpose(0, 1).unsqueeze(0)
    tv = torch.tensor(V).view(n, H, d // H).transpose(0, 1).unsqueeze(0)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, scale=sc)
    assert np.allclose(out, ref.reshape(d).numpy(), atol=1e-13)


def test_hybrid_equivalence_against_torch_projection():
    """hidden(X) == KV(K = X W_K^T + b_K, V = X W_V^T + b_V) (north_star invariant),
    with the twin K/V computed by torch float64 rather than by the oracle."""
    d, n, H = 32, 21, 2
    X, W, b, q = _rand((n, d), 23), _rand((2 * d, d), 24, 0.2), _rand(2 * d, 25, 0.02), _rand(d, 26)
    tX, tW, tb = torch.tensor(X), torch.tensor(W), torch.tensor(b)
    KV = torch.nn.functional.linear(tX, tW, tb).numpy()
    oh, lh = O.decode_batch([{"mode": 1, "q": q, "X": X}], W, H, 0.25, b)
    ok, lk = O.decode_batch([{"mode": 0, "q": q, "K": KV[:, :d], "V": KV[:, d:]}], W, H, 0.25)
    assert np.allclose(oh, ok, atol=1e-13) and np.allclose(lh, lk, atol=1e-13)


def test_lse_matches_scipy_logsumexp():
    from scipy.special import logsumexp
    d, n, H, sc = 16, 40, 4, 0.7
    q, K, V = _rand(d, 27), _rand((n, d), 28), _rand((n, d), 29)
    _, lse = O.attend(q, K, V, H, sc)
    for h in range(H):
        c = slice(h * 4, (h + 1) * 4)
        assert abs(lse[h] - logsumexp(sc * K[:, c] @ q[c])) < 1e-13


def test_order_of_tokens_is_irrelevant():
    """Attention without positional terms is permutation-invariant over keys (block
    indirection may store tokens anywhere; SURVEY §8(c) 'Block indirection')."""
    d, n = 16, 25
    q, K, V = _rand(d, 30), _rand((n, d), 31), _rand((n, d), 32)
    p = np.random.default_rng(33).permutation(n)
    a, la = O.attend(q, K, V, 2, 0.4)
    b, lb = O.attend(q, K[p], V[p], 2, 0.4)
    assert np.allclose(a, b, atol=1e-14) and np.allclose(la, lb, atol=1e-14)


def test_max_rel_err_definition():
    ref = np.array([[1.0, -2.0, 0.5, 0.25]])
    gpu = ref + np.array([[0.0, 0.02, 0.0, 0.0025]])
    # head 0 cols (1,-2): 0.02/2 = 0.01 ; head 1 cols (0.5,0.25): 0.0025/0.5 = 0.005
    assert abs(O.max_rel_err(gpu, ref, 2) - 0.01) < 1e-15


def test_zero_context_is_rejected():
    with pytest.raises(AssertionError):
        O.attend(np.zeros(4), np.zeros((0, 4)), np.zeros((0, 4)), 1, 1.0)


# ---------------------------------------------------------------- attention layer (f1)
def test_layer_identity_maps_reduce_to_decode():
    """W_Q = I, W_O = I, W_KV = [I; I]: q = x_t, k_t = v_t = x_t, y = o — the layer is the
    decode step over the cache extended by x_t (hidden) or (x_t, x_t) (KV)."""
    d, H, n = 12, 3, 9
    I = np.eye(d)
    x = _rand(d, 40)
    X = _rand((n, d), 41)
    y, q, lse, ctx = O.attention_layer(x, {"mode": 1, "X": X}, I, np.vstack([I, I]), I, H, 0.5)
    assert np.array_equal(q, x)
    o, l = O.attend(x, np.vstack([X, x]), np.vstack([X, x]), H, 0.5)
    assert np.allclose(y, o, atol=1e-14) and np.allclose(lse, l, atol=1e-14)
    K, V = _rand((n, d), 42), _rand((n, d), 43)
    y2, _, _, ctx2 = O.attention_layer(x, {"mode": 0, "K": K, "V": V}, I, np.vstack([I, I]), I, H, 0.5)
    assert np.array_equal(ctx2["K"][-1], x) and np.array_equal(ctx2["V"][-1], x)


def test_layer_hidden_equals_kv_twin_and_matches_torch():
    """hidden(X + x_t) == KV(K, V projected from X + x_t) through the whole layer, and the
    layer equals a torch float64 composition (linear -> SDPA -> linear)."""
    d, H, n = 16, 2, 11
    W_Q, W_KV, W_O = _rand((d, d), 44, 0.3), _rand((2 * d, d), 45, 0.3), _rand((d, d), 46, 0.3)
    b_Q, b_KV, b_O = _rand(d, 47, 0.1), _rand(2 * d, 48, 0.1), _rand(d, 49, 0.1)
    x, X = _rand(d, 50), _rand((n, d), 51)
    yh, qh, lh, _ = O.attention_layer(x, {"mode": 1, "X": X}, W_Q, W_KV, W_O, H, 0.25, b_Q, b_KV, b_O)
    KV = X @ W_KV.T + b_KV
    yk, qk, lk, _ = O.attention_layer(x, {"mode": 0, "K": KV[:, :d], "V": KV[:, d:]}, W_Q, W_KV, W_O, H, 0.25,
                                      b_Q, b_KV, b_O)
    assert np.allclose(yh, yk, atol=1e-12) and np.allclose(lh, lk, atol=1e-12)
    tX = torch.tensor(np.vstack([X, x]))
    kv = torch.nn.functional.linear(tX, torch.tensor(W_KV), torch.tensor(b_KV))
    q = torch.nn.functional.linear(torch.tensor(x), torch.tensor(W_Q), torch.tensor(b_Q))
    dh = d // H
    att = torch.nn.functional.scaled_dot_product_attention(
        q.view(1, H, 1, dh), kv[:, :d].view(-1, H, dh).transpose(0, 1).unsqueeze(0),
        kv[:, d:].view(-1, H, dh).transpose(0, 1).unsqueeze(0), scale=0.25).reshape(d)
    y_t = torch.nn.functional.linear(att, torch.tensor(W_O), torch.tensor(b_O)).numpy()
    assert np.allclose(yh, y_t, atol=1e-12)


# ---------------------------------------------------------------- prefill (f3)
def test_prefill_first_row_and_last_row_consistency():
    """Row 0 attends only to itself (o_0 = v_0); the last row equals the decode-layer step
    with the first L-1 tokens cached (the current token attends to all previous and itself)."""
    d, H, L = 16, 2, 9
    W_Q, W_KV, W_O = _rand((d, d), 60, 0.3), _rand((2 * d, d), 61, 0.3), _rand((d, d), 62, 0.3)
    b_Q, b_KV, b_O = _rand(d, 63, 0.1), _rand(2 * d, 64, 0.1), _rand(d, 65, 0.1)
    X = _rand((L, d), 66)
    Y, K, V = O.prefill_layer(X, W_Q, W_KV, W_O, H, 0.3, b_Q, b_KV, b_O)
    assert np.allclose(Y[0], W_O @ V[0] + b_O, atol=1e-13)
    y_last, _, _, _ = O.attention_layer(X[-1], {"mode": 1, "X": X[:-1]}, W_Q, W_KV, W_O, H, 0.3, b_Q, b_KV, b_O)
    assert np.allclose(Y[-1], y_last, atol=1e-12)


def test_prefill_matches_torch_causal_sdpa():
    d, H, L = 24, 3, 13
    W_Q, W_KV, W_O = _rand((d, d), 67, 0.3), _rand((2 * d, d), 68, 0.3), _rand((d, d), 69, 0.3)
    X = _rand((L, d), 70)
    Y, _, _ = O.prefill_layer(X, W_Q, W_KV, W_O, H, 0.4)
    tX = torch.tensor(X)
    q = (tX @ torch.tensor(W_Q).T).view(L, H, d // H).transpose(0, 1)
    kv = tX @ torch.tensor(W_KV).T
    k = kv[:, :d].view(L, H, d // H).transpose(0, 1)
    v = kv[:, d:].view(L, H, d // H).transpose(0, 1)
    att = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=0.4)
    y_t = att.transpose(0, 1).reshape(L, d) @ torch.tensor(W_O).T
    assert np.allclose(Y, y_t.numpy(), atol=1e-12)


# ---------------------------------------------------------------- RoPE (f4)
def test_rope_identity_norm_and_relative_position():
    """Position 0 is the identity; rotations preserve per-head norms; the score of a
    rotated pair depends only on the position difference (the defining RoPE property)."""
    d, H, theta = 32, 2, 10000.0
    U = _rand((5, d), 80)
    assert np.array_equal(O.rope(U, [0] * 5, theta, H), U)
    R = O.rope(U, [3, 17, 1000, 123456, 7], theta, H)
    for h in range(H):
        c = slice(h * 16, (h + 1) * 16)
        assert np.allclose(np.linalg.norm(R[:, c], axis=1), np.linalg.norm(U[:, c], axis=1), atol=1e-12)
    q, k = _rand((1, d), 81), _rand((1, d), 82)
    s1 = O.rope(q, [10], theta, H) @ O.rope(k, [4], theta, H).T
    s2 = O.rope(q, [1006], theta, H) @ O.rope(k, [1000], theta, H).T
    assert np.allclose(s1, s2, atol=1e-10)


def test_rope_matches_hf_rotate_half_in_torch():
    """Library-style formula (HF LlamaRotaryEmbedding + rotate_half) in torch float64."""
    d, H, theta, n = 24, 2, 500000.0, 9
    dh = d // H
    U = _rand((n, d), 83)
    pos = torch.arange(n, dtype=torch.float64) * 37
    inv = 1.0 / (theta ** (torch.arange(0, dh, 2, dtype=torch.float64) / dh))
    emb = torch.cat([pos[:, None] * inv[None, :]] * 2, dim=-1)
    u = torch.tensor(U).view(n, H, dh)
    rot = torch.cat([-u[..., dh // 2:], u[..., :dh // 2]], dim=-1)
    ref = (u * emb.cos()[:, None, :] + rot * emb.sin()[:, None, :]).reshape(n, d)
    assert np.allclose(O.rope(U, pos.numpy(), theta, H), ref.numpy(), atol=1e-12)


def test_rope_hidden_equals_rotated_kv_twin():
    """hidden(X) with RoPE == KV twin holding rotated keys (P:269 + rotation at position j)."""
    d, H, n, theta = 16, 2, 12, 10000.0
    W, X, q = _rand((2 * d, d), 84, 0.3), _rand((n, d), 85), _rand(d, 86)
    K, V = O.hidden_request_kv(X, W)
    Kr = O.rope(K, np.arange(n), theta, H)
    oh, lh = O.decode_batch([{"mode": 1, "q": q, "X": X}], W, H, 0.3, rope_theta=theta)
    ok, lk = O.decode_batch([{"mode": 0, "q": q, "K": Kr, "V": V}], W, H, 0.3)
    assert np.allclose(oh, ok, atol=1e-13) and np.allclose(lh, lk, atol=1e-13)


# ---------------------------------------------------------------- pre-attention LayerNorm (f1 option)
def test_layer_norm_matches_torch_and_is_shift_invariant():
    """LN against torch.nn.functional.layer_norm in float64 (library routine); exact
    invariance to adding a constant to a row; gamma = 1, beta = 0 gives mean 0 and
    variance var / (var + eps) per row."""
    rs = np.random.default_rng(5)
    X = rs.normal(size=(7, 48)) * 3.0 + 2.0
    g, b = 1 + 0.1 * rs.normal(size=48), 0.02 * rs.normal(size=48)
    ref = torch.nn.functional.layer_norm(torch.from_numpy(X), (48,), torch.from_numpy(g), torch.from_numpy(b), 1e-5)
    assert np.allclose(O.layer_norm(X, g, b, 1e-5), ref.numpy(), rtol=0, atol=1e-12)
    assert np.allclose(O.layer_norm(X + 5.0, g, b), O.layer_norm(X, g, b), rtol=0, atol=1e-12)
    U = O.layer_norm(X, np.ones(48), None, 1e-5)
    var = X.var(axis=1)
    assert np.allclose(U.mean(axis=1), 0, atol=1e-12)
    assert np.allclose(U.var(axis=1), var / (var + 1e-5), rtol=1e-12)


def test_layer_with_ln_is_layer_on_normalised_input():
    """attention_layer / prefill_layer with ln = the same layers fed LN(x) (the hidden cache
    holds u = LN(x), reading R15), for both cache modes."""
    rs = np.random.default_rng(6)
    d, H, n = 32, 2, 9
    Wq, Wkv, Wo = rs.normal(size=(d, d)) / 6, rs.normal(size=(2 * d, d)) / 6, rs.normal(size=(d, d)) / 6
    g, b = 1 + 0.1 * rs.normal(size=d), 0.02 * rs.normal(size=d)
    X = rs.normal(size=(n, d)) * 2 + 1
    ln = (g, b, 1e-5)
    U = O.layer_norm(X, *ln)
    for mode in (0, 1):
        if mode == 1:
            cache = {"mode": 1, "X": U[:-1]}
        else:
            KV = U[:-1] @ Wkv.T
            cache = {"mode": 0, "K": KV[:, :d], "V": KV[:, d:]}
        y1, q1, l1, _ = O.attention_layer(X[-1], cache, Wq, Wkv, Wo, H, 0.25, ln=ln)
        y2, q2, l2, _ = O.attention_layer(U[-1], cache, Wq, Wkv, Wo, H, 0.25)
        assert np.array_equal(y1, y2) and np.array_equal(l1, l2)
    Y1, _, _ = O.prefill_layer(X, Wq, Wkv, Wo, H, 0.25, ln=ln)
    Y2, _, _ = O.prefill_layer(U, Wq, Wkv, Wo, H, 0.25)
    assert np.array_equal(Y1, Y2)
    # and the LN really changes the layer for this input
    Y3, _, _ = O.prefill_layer(X, Wq, Wkv, Wo, H, 0.25)
    assert np.abs(Y1 - Y3).max() > 1e-3


# ---------------------------------------------------------------- the per-head sampling path
def _sampling_cases():
    from synth.configs import LayerShape, Workload
    small = LayerShape("pin-small", 64, 4, 16)
    gqa = LayerShape("pin-gqa", 64, 8, 8, 2)      # 8 query heads over 2 K/V heads
    n = [1, 17, 40, 33]
    modes = [C.MODE_HIDDEN, C.MODE_KV, C.MODE_HIDDEN, C.MODE_HIDDEN]
    return [
        ("tiny-f32", C.tiny(bias=False), 0.0),
        ("tiny-f32-bias", C.tiny(bias=True), 0.0),
        ("small-bf16-bias", Workload("pin-bf16", small, 16, "bf16", 11, n, modes, [5, 6, 7, 8], True), 0.0),
        ("small-bf16-rope", Workload("pin-rope", small, 16, "bf16", 12, n, modes, [1, 2, 3, 4], True), 10000.0),
        ("small-bf16-peaky", Workload("pin-peaky", small, 16, "bf16", 13, n, modes, [1, 2, 3, 4], True,
                                      q_scale=4.0), 0.0),
        ("small-gqa-bias", Workload("pin-gqa", gqa, 16, "bf16", 14, n, modes, [1, 2, 3, 4], True), 0.0),
        ("small-gqa-rope", Workload("pin-gqa-rope", gqa, 16, "bf16", 15, n, modes, [1, 2, 3, 4], True), 500000.0),
    ]


@pytest.mark.parametrize("name,w,theta", _sampling_cases(), ids=[c[0] for c in _sampling_cases()])
def test_per_head_sampling_equals_decode_batch(name, w, theta):
    """The per-head path every full-size GPU check goes through (tests/hc_testlib.oracle_request
    -> hc_oracle.head_output, which rebuilds only head h's dh columns of K and V) equals the
    Decimal-pinned decode_batch on every head, to 1e-13 — for all heads at once and for
    scattered head subsets, with bias, RoPE and a peaky query (Eq. 1-3)."""
    from tests import hc_testlib as T
    d, H = w.shape.d, w.shape.H
    W, b = w.w_kv(), w.b_kv()
    for i in range(len(w.n)):
        q = w.q(i).double().numpy()
        if w.modes[i] == C.MODE_KV:
            K, V = w.kv(i)
            req = {"mode": 0, "q": q, "K": K, "V": V}
        else:
            req = {"mode": 1, "q": q, "X": w.x(i)}
        ref, lref = O.decode_batch([req], W, H, w.scale, b, rope_theta=theta, n_kv_heads=w.shape.n_kv)
        for heads in (None, [H - 1, 0], [1]):
            o, l = T.oracle_request(w, i, heads, rope_theta=theta)
            hs = list(range(H)) if heads is None else heads
            dh = d // H
            want = np.concatenate([ref[0, h * dh:(h + 1) * dh] for h in hs])
            assert np.allclose(o, want, rtol=0, atol=1e-13 * max(1.0, np.abs(want).max())), (name, i, heads)
            assert np.allclose(l, lref[0, hs], rtol=0, atol=1e-12), (name, i, heads)


def test_head_output_against_decimal_bruteforce():
    """head_output itself against 40-digit Decimal on one hidden request with a bias: k = W_K,h x
    + b_K,h, v = W_V,h x + b_V,h, softmax with the given scale (catches swapped biases, a
    wrong scale or a transposed W in the per-head path)."""
    rs = np.random.default_rng(3)
    n, d, dh = 7, 12, 4
    X = rs.normal(size=(n, d))
    WK, WV = rs.normal(size=(dh, d)), rs.normal(size=(dh, d))
    bK, bV = rs.normal(size=dh), rs.normal(size=dh) + 3.0
    q = rs.normal(size=dh)
    scale = 0.37
    o, l = O.head_output(q, X, WK, WV, scale, bK, bV)
    Xd = [[Decimal(repr(float(v))) for v in row] for row in X]
    Kd = _dec_recon(Xd, _dec_matrix(torch.tensor(WK)), [Decimal(repr(float(v))) for v in bK])
    Vd = _dec_recon(Xd, _dec_matrix(torch.tensor(WV)), [Decimal(repr(float(v))) for v in bV])
    o_ref, l_ref = _dec_attend(q, Kd, Vd, 1, scale)
    assert np.allclose(o, [float(x) for x in o_ref], rtol=0, atol=1e-13)
    assert abs(l - float(l_ref[0])) < 1e-13


def test_layer_norm_store_rounding_is_one_bf16_rounding():
    """R16: store="bf16" is exactly one round-to-nearest of the fp64 LN to bf16 — every value is
    representable in bf16 (8 significant bits) and within half an ulp of the unrounded LN,
    and rounding is idempotent."""
    rs = np.random.default_rng(8)
    X = rs.normal(size=(5, 64)) * 2.5 + 1.0
    g, b = 1 + 0.1 * rs.normal(size=64), 0.02 * rs.normal(size=64)
    U = O.layer_norm(X, g, b, 1e-5)
    Us = O.layer_norm(X, g, b, 1e-5, store="bf16")
    m, e = np.frexp(Us)
    assert np.array_equal(m * 256, np.round(m * 256))          # 8-bit significand
    ulp = np.ldexp(1.0, np.frexp(U)[1] - 8)
    assert np.all(np.abs(Us - U) <= 0.5 * ulp + 1e-300)
    again = torch.from_numpy(Us).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(again, Us)                             # idempotent
    assert not np.array_equal(Us, U)                             # and it did round



# ---------------------------------------------------------------- grouped-query attention (f4 (i), R18)
def _gqa_tiny(seed=21, bias=True):
    from synth.configs import LayerShape, Workload
    sh = LayerShape("pin-gqa-tiny", 32, 4, 8, 2)
    return Workload("gqa-tiny", sh, 4, "f32", seed, [9, 1, 6, 12], [C.MODE_KV, C.MODE_HIDDEN, C.MODE_HIDDEN,
                                                                   C.MODE_KV], [0, 1, 2, 3], bias)


def test_gqa_vs_decimal_bruteforce():
    """GQA decode (query head h reads K/V head h // G) against a 40-digit Decimal brute force
    that writes the head mapping out by hand: tiny shape, 4 query heads over 2 K/V heads,
    both cache modes, with bias."""
    w = _gqa_tiny()
    d, H, dh, Hk = w.shape.d, w.shape.H, w.shape.dh, w.shape.n_kv
    dk, G = Hk * dh, H // Hk
    W, b = w.w_kv(), w.b_kv()
    Wd = _dec_matrix(W.double())
    bd = [Decimal(repr(float(v))) for v in b.tolist()]
    getcontext().prec = 40
    for i in range(4):
        q = w.q(i).double().numpy()
        if w.modes[i] == C.MODE_KV:
            K, V = w.kv(i)
            Kd, Vd = _dec_matrix(K.double()), _dec_matrix(V.double())
            req = {"mode": 0, "q": q, "K": K, "V": V}
        else:
            Xd = _dec_matrix(w.x(i).double())
            Kd, Vd = _dec_recon(Xd, Wd[:dk], bd[:dk]), _dec_recon(Xd, Wd[dk:], bd[dk:])
            req = {"mode": 1, "q": q, "X": w.x(i)}
        out, lse = O.decode_batch([req], W, H, w.scale, b, n_kv_heads=Hk)
        sc = Decimal(repr(w.scale))
        for h in range(H):
            hk = h // G
            s = [sc * sum(Decimal(repr(float(q[h * dh + c]))) * Kd[j][hk * dh + c] for c in range(dh))
                 for j in range(len(Kd))]
            m = max(s)
            e = [(x - m).exp() for x in s]
            z = sum(e)
            for c in range(dh):
                ref = float(sum(e[j] / z * Vd[j][hk * dh + c] for j in range(len(Kd))))
                assert abs(out[0, h * dh + c] - ref) <= 1e-13 * max(1.0, abs(ref))
            assert abs(lse[0, h] - float(m + z.ln())) <= 1e-13


def test_gqa_equals_multihead_with_repeated_kv_heads():
    """Closed form: GQA over Hk heads = multi-head attention over K/V whose heads are repeated
    G times (repeat_interleave over heads), for KV and hidden requests (W_K, W_V rows repeated)."""
    rs = np.random.default_rng(22)
    n, H, Hk, dh = 11, 6, 2, 4
    d, dk, G = H * dh, Hk * dh, H // Hk
    q, K, V = rs.normal(size=d), rs.normal(size=(n, dk)), rs.normal(size=(n, dk))
    rep = lambda M: np.repeat(M.reshape(M.shape[0], Hk, dh), G, axis=1).reshape(M.shape[0], d)
    o1, l1 = O.attend(q, K, V, H, 0.3, n_kv_heads=Hk)
    o2, l2 = O.attend(q, rep(K), rep(V), H, 0.3)
    assert np.allclose(o1, o2, rtol=0, atol=1e-14) and np.allclose(l1, l2, rtol=0, atol=1e-14)
    X, W, bb = rs.normal(size=(n, d)), rs.normal(size=(2 * dk, d)), rs.normal(size=2 * dk)
    Wrep = np.concatenate([rep(W[:dk].T).T, rep(W[dk:].T).T])
    brep = np.concatenate([rep(bb[None, :dk])[0], rep(bb[None, dk:])[0]])
    a1, _ = O.decode_batch([{"mode": 1, "q": q, "X": X}], W, H, 0.3, bb, n_kv_heads=Hk)
    a2, _ = O.decode_batch([{"mode": 1, "q": q, "X": X}], Wrep, H, 0.3, brep)
    assert np.allclose(a1, a2, rtol=0, atol=1e-12)


def test_gqa_matches_torch_sdpa_enable_gqa():
    """Library routine: torch scaled_dot_product_attention(enable_gqa=True) in float64 with one
    query per request; and the hybrid equivalence hidden(X) = KV(X W_K^T + b_K, X W_V^T + b_V)."""
    rs = np.random.default_rng(23)
    n, H, Hk, dh = 13, 8, 2, 16
    d, dk = H * dh, Hk * dh
    q, X = rs.normal(size=d), rs.normal(size=(n, d))
    W, bb = rs.normal(size=(2 * dk, d)) / np.sqrt(d), rs.normal(size=2 * dk) * 0.1
    K, V = X @ W[:dk].T + bb[:dk], X @ W[dk:].T + bb[dk:]
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q).view(1, H, 1, dh), torch.from_numpy(K).view(n, Hk, dh).transpose(0, 1)[None],
        torch.from_numpy(V).view(n, Hk, dh).transpose(0, 1)[None], scale=0.25, enable_gqa=True)
    o_kv, _ = O.decode_batch([{"mode": 0, "q": q, "K": K, "V": V}], W, H, 0.25, bb, n_kv_heads=Hk)
    o_h, _ = O.decode_batch([{"mode": 1, "q": q, "X": X}], W, H, 0.25, bb, n_kv_heads=Hk)
    assert np.allclose(o_kv[0], ref.reshape(-1).numpy(), rtol=0, atol=1e-12)
    assert np.allclose(o_h[0], o_kv[0], rtol=0, atol=1e-12)


def test_gqa_layers_equal_multihead_layers_with_repeated_kv_weights():
    """attention_layer / prefill_layer under GQA = the multi-head layers whose W_K, W_V (and
    biases) repeat each K/V head's rows G times — for both cache modes, with RoPE."""
    rs = np.random.default_rng(24)
    H, Hk, dh, n = 4, 2, 8, 7
    d, dk, G = H * dh, Hk * dh, H // Hk
    Wq, Wo = rs.normal(size=(d, d)) / 6, rs.normal(size=(d, d)) / 6
    Wkv, bkv = rs.normal(size=(2 * dk, d)) / 6, rs.normal(size=2 * dk) * 0.1
    rep_rows = lambda M: np.repeat(M.reshape(Hk, dh, -1), G, axis=0).reshape(d, -1)
    Wrep = np.concatenate([rep_rows(Wkv[:dk]), rep_rows(Wkv[dk:])])
    brep = np.concatenate([rep_rows(bkv[:dk, None])[:, 0], rep_rows(bkv[dk:, None])[:, 0]])
    X = rs.normal(size=(n, d))
    for theta in (0.0, 10000.0):
        for mode in (0, 1):
            if mode == 1:
                c1 = c2 = {"mode": 1, "X": X[:-1]}
            else:
                KV = X[:-1] @ Wkv.T + bkv
                K = O.rope(KV[:, :dk], np.arange(n - 1), theta, Hk)
                c1 = {"mode": 0, "K": K, "V": KV[:, dk:]}
                c2 = {"mode": 0, "K": np.repeat(K.reshape(n - 1, Hk, dh), G, axis=1).reshape(n - 1, d),
                      "V": np.repeat(KV[:, dk:].reshape(n - 1, Hk, dh), G, axis=1).reshape(n - 1, d)}
            y1, _, l1, _ = O.attention_layer(X[-1], c1, Wq, Wkv, Wo, H, 0.3, b_KV=bkv, rope_theta=theta)
            y2, _, l2, _ = O.attention_layer(X[-1], c2, Wq, Wrep, Wo, H, 0.3, b_KV=brep, rope_theta=theta)
            assert np.allclose(y1, y2, rtol=0, atol=1e-12) and np.allclose(l1, l2, rtol=0, atol=1e-12)
        Y1, _, _ = O.prefill_layer(X, Wq, Wkv, Wo, H, 0.3, b_KV=bkv, rope_theta=theta)
        Y2, _, _ = O.prefill_layer(X, Wq, Wrep, Wo, H, 0.3, b_KV=brep, rope_theta=theta)
        assert np.allclose(Y1, Y2, rtol=0, atol=1e-12)
