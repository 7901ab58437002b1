"""fp64 CPU ORACLE for one decode-step attention layer over the hybrid cache.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import or call anything under `oracle/`.
The product path (paper_2504_07494_b200/) never imports it and shares no code with it.

What it computes (§2.1, Eq. 1-3; §3.1 "Opportunity I"):
for each request i in the decode batch, with n_i >= 1 cached tokens INCLUDING the
current one (the current token "attends to ... itself"):

  1. K/V source.  KV mode (beta_i = 0): k_j, v_j are read from the cache.
     Hidden mode (beta_i = 1): the cache holds the layer input x_j and
         k_j = W_K x_j (+ b_K),   v_j = W_V x_j (+ b_V)              (Eq. 1)
     for every cached j ("transform the cached input hidden vectors ... to required key
     and value vectors").  No pre-projection normalisation: the paper specifies
     none (reading R4); the bias is optional (reading R4).
  2. Per head h (columns h*dh .. h*dh+dh-1 of d; reading R1):
         s_j = scale * q_h . k_{j,h}                                 (Eq. 2)
         a_j = exp(s_j - max s) / sum_m exp(s_m - max s)              (Eq. 2)
         o_h = sum_j a_j v_{j,h}                                     (Eq. 3, P:131-133;
                                                v_i in the paper is a typo for v_j, R2)
     out_i = concat_h o_h  (before W_o, reading R3);  lse_{i,h} = max s + ln sum exp(s - max s).

Everything is float64; inputs stored in bf16/fp32 are widened exactly.  The oracle does
NOT round reconstructed K/V to the storage precision (reading R9): the GPU's rounding
is part of the error the tolerance covers.

Pins (tests/test_oracle_pins.py): 40-digit Decimal brute force, closed forms (W = I,
permutation W, n = 1, q = 0, V = 1, bias shift), torch float64 SDPA, hybrid equivalence,
softmax rows summing to 1.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np


def _f64(a) -> np.ndarray:
    """Exact widening of a torch / numpy array to float64."""
    if hasattr(a, "detach"):
        a = a.detach().cpu().to(dtype=__import__("torch").float64).numpy()
    return np.asarray(a, dtype=np.float64)


def rope(U, positions, theta: float, n_heads: int):
    """Rotary position embedding (NEXT row f4; the LLaMA / Yi models of §6.6), NeoX
    "rotate_half" convention, fp64: per head u = [u1, u2] (halves of dh),
        u' = [u1 cos(p w) - u2 sin(p w),  u2 cos(p w) + u1 sin(p w)],  w_c = theta^(-2c/dh).
    U: [n, d] rows at token positions `positions` [n].  theta = 0 returns U unchanged."""
    U = _f64(U)
    if theta == 0:
        return U
    n, d = U.shape
    dh = d // n_heads
    half = dh // 2
    w = theta ** (-2.0 * np.arange(half) / dh)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * w[None, :]
    cs, sn = np.cos(ang), np.sin(ang)
    out = U.copy()
    for h in range(n_heads):
        a = U[:, h * dh:h * dh + half]
        b = U[:, h * dh + half:(h + 1) * dh]
        out[:, h * dh:h * dh + half] = a * cs - b * sn
        out[:, h * dh + half:(h + 1) * dh] = b * cs + a * sn
    return out


def reconstruct_kv(X, W_K, W_V, b_K=None, b_V=None):
    """Eq. 1 applied to every cached hidden state:
    K = X W_K^T (+ b_K), V = X W_V^T (+ b_V).  X: [n, d]; W_K, W_V: [d, d] with
    k = W_K x (rows of W are output features)."""
    X, W_K, W_V = _f64(X), _f64(W_K), _f64(W_V)
    K = X @ W_K.T
    V = X @ W_V.T
    if b_K is not None:
        K = K + _f64(b_K)[None, :]
    if b_V is not None:
        V = V + _f64(b_V)[None, :]
    return K, V


def attend(q, K, V, n_heads: int, scale: float, return_probs: bool = False, n_kv_heads: Optional[int] = None):
    """Eq. 2-3 for ONE decode query over n cached tokens, per head.
    q: [d]; K, V: [n, Hk*dh].  Returns out [d], lse [H] (and probabilities [H, n]).
    n_kv_heads = Hk < H: grouped-query attention (the LLaMA-3 / Yi models of §6.6, P:645;
    DESIGN R18): query head h reads key/value head h // (H / Hk).  Hk = H (default) is Eq. 2-3
    per head exactly as written."""
    q, K, V = _f64(q), _f64(K), _f64(V)
    n = K.shape[0]
    d = q.shape[0]
    assert n >= 1, "n_i >= 1: the current token is part of the context (P:135)"
    dh = d // n_heads
    Hk = n_heads if n_kv_heads is None else n_kv_heads
    assert n_heads % Hk == 0 and K.shape[1] == Hk * dh and V.shape[1] == Hk * dh
    G = n_heads // Hk
    out = np.empty(d)
    lse = np.empty(n_heads)
    probs = np.empty((n_heads, n))
    for h in range(n_heads):
        c = slice(h * dh, (h + 1) * dh)
        ck = slice((h // G) * dh, (h // G + 1) * dh)   # this query head's key/value head
        s = scale * (K[:, ck] @ q[c])         # s_j = q_h . k_{j,h} / sqrt(.)
        m = s.max()
        e = np.exp(s - m)
        l = e.sum()
        a = e / l                              # a_j, Eq. 2
        out[c] = a @ V[:, ck]                  # sum_j a_j v_{j,h}, Eq. 3 (pre-W_o)
        lse[h] = m + np.log(l)
        probs[h] = a
    if return_probs:
        return out, lse, probs
    return out, lse


def hidden_request_kv(X, W_KV, b_KV=None):
    """Split the stacked [2 Dk, d] W_KV = [W_K; W_V] (and [2 Dk] bias; Dk = d for multi-head,
    Hk*dh under GQA) and rebuild K, V [n, Dk]."""
    W_KV = _f64(W_KV)
    dk = W_KV.shape[0] // 2
    bK = bV = None
    if b_KV is not None:
        b = _f64(b_KV)
        bK, bV = b[:dk], b[dk:]
    return reconstruct_kv(X, W_KV[:dk], W_KV[dk:], bK, bV)


def decode_batch(requests: Sequence[dict], W_KV, n_heads: int, scale: float, b_KV=None, rope_theta: float = 0.0,
                 n_kv_heads: Optional[int] = None):
    """Hybrid-cache decode step for a batch.  Each request dict has 'q' [d] and either
    'mode' 0 with 'K', 'V' [n, Dk] or 'mode' 1 with 'X' [n, d] (Dk = Hk*dh, = d unless GQA).
    With RoPE, rebuilt keys are rotated at their token positions 0..n-1 (cached KV-mode keys
    are stored rotated; q is given rotated).  Returns out [n_req, d], lse [n_req, H]."""
    Hk = n_heads if n_kv_heads is None else n_kv_heads
    outs, lses = [], []
    for r in requests:
        if r["mode"] == 1:
            K, V = hidden_request_kv(r["X"], W_KV, b_KV)
            K = rope(K, np.arange(K.shape[0]), rope_theta, Hk)
        else:
            K, V = r["K"], r["V"]
        o, l = attend(r["q"], K, V, n_heads, scale, n_kv_heads=Hk)
        outs.append(o)
        lses.append(l)
    return np.stack(outs), np.stack(lses)


def head_output(q_h, X, W_K_h, W_V_h, scale: float, b_K_h=None, b_V_h=None):
    """One (request, head) of a hidden-mode request, rebuilding only that head's
    dh columns (the same Eq. 1-3 restricted to head h; used to sample large configs)."""
    K, V = reconstruct_kv(X, W_K_h, W_V_h, b_K_h, b_V_h)
    o, l = attend(q_h, K, V, 1, scale)
    return o, l[0]


def layer_norm(X, gamma, beta=None, eps: float = 1e-5, store: Optional[str] = None):
    """Pre-attention LayerNorm of OPT-style layers (the paper's Eq. 1
    specifies none, DESIGN R4/R15): per row, (x - mean) / sqrt(var + eps) * gamma + beta
    with the population variance over the d features.
    store="bf16" (DESIGN R16): u is a STORED vector — the hidden cache holds it (R15) in the
    storage precision (R9), and it is the input Eq. 1 multiplies — so the result is rounded
    once to bf16 (round-to-nearest-even), exactly as the oracle takes stored bf16 x as given."""
    X = _f64(X)
    mu = X.mean(axis=-1, keepdims=True)
    var = ((X - mu) ** 2).mean(axis=-1, keepdims=True)
    Y = (X - mu) / np.sqrt(var + eps) * _f64(gamma)
    Y = Y + (0.0 if beta is None else _f64(beta))
    if store == "bf16":
        import torch
        Y = torch.from_numpy(np.ascontiguousarray(Y)).to(torch.bfloat16).to(torch.float64).numpy()
    return Y


def attention_layer(x_t, cache: dict, W_Q, W_KV, W_O, n_heads: int, scale: float,
                    b_Q=None, b_KV=None, b_O=None, rope_theta: float = 0.0, ln=None):
    """One attention layer for one decode step of one request (NEXT row f1):
    q = W_Q x_t (+b_Q) and, for the current token, k, v = W_K x_t, W_V x_t (+b)  (Eq. 1,
    P:121-125); the current token joins the context: KV mode appends (k, v) to
    the cached K, V; hidden mode appends x_t to the cached X and rebuilds K, V from all of X
    (P:269); then Eq. 2-3 with the output map y = W_O o (+b_O) (Eq. 3).
    cache = {'mode': 0, 'K': [n-1, d], 'V': [n-1, d]} or {'mode': 1, 'X': [n-1, d]}.
    ln = (gamma, beta, eps[, store]) or None: the projections see u_t = LN(x_t), and a hidden
    cache holds u (the vector Eq. 1 multiplies; reading R15) — cache['X'] rows are stored u's;
    store = "bf16" rounds u_t to the storage precision (reading R16).
    Returns y [d], q [d], lse [H], and the context the attention saw (dict)."""
    x_t, W_Q, W_O = _f64(x_t), _f64(W_Q), _f64(W_O)
    if ln is not None:
        x_t = layer_norm(x_t[None, :], *ln)[0]
    W_KV = _f64(W_KV)
    d = x_t.shape[0]
    dk = W_KV.shape[0] // 2                       # K/V row width (d, or Hk*dh under GQA, R18)
    Hk = n_heads * dk // d
    q = W_Q @ x_t + (0.0 if b_Q is None else _f64(b_Q))
    if cache["mode"] == 1:
        X = np.concatenate([_f64(cache["X"]).reshape(-1, d), x_t[None, :]])
        pos = X.shape[0] - 1
        K, V = hidden_request_kv(X, W_KV, b_KV)
        K = rope(K, np.arange(X.shape[0]), rope_theta, Hk)
        ctx = {"mode": 1, "X": X}
    else:
        kv = W_KV @ x_t + (0.0 if b_KV is None else _f64(b_KV))
        pos = _f64(cache["K"]).reshape(-1, dk).shape[0]
        kv[:dk] = rope(kv[None, :dk], [pos], rope_theta, Hk)[0]
        K = np.concatenate([_f64(cache["K"]).reshape(-1, dk), kv[None, :dk]])
        V = np.concatenate([_f64(cache["V"]).reshape(-1, dk), kv[None, dk:]])
        ctx = {"mode": 0, "K": K, "V": V}
    q = rope(q[None, :], [pos], rope_theta, n_heads)[0]
    o, lse = attend(q, K, V, n_heads, scale, n_kv_heads=Hk)
    y = W_O @ o + (0.0 if b_O is None else _f64(b_O))
    return y, q, lse, ctx


def prefill_layer(X, W_Q, W_KV, W_O, n_heads: int, scale: float, b_Q=None, b_KV=None, b_O=None,
                  rope_theta: float = 0.0, ln=None):
    """Prefill of one request's L new tokens (NEXT row f3): q, k, v of every
    token (Eq. 1), then for each position i causal attention over tokens j <= i (Eq. 2-3,
    P:127-135: "attending to all of the preceding tokens and itself") and the output map.
    Returns Y [L, d] and the K, V [L, d] the cache must hold (KV mode) — hidden mode caches X
    (with ln = (gamma, beta, eps): every row is LN(x) first and the hidden cache holds it)."""
    X, W_Q, W_O = _f64(X), _f64(W_Q), _f64(W_O)
    if ln is not None:
        X = layer_norm(X, *ln)
    L, d = X.shape
    Q = X @ W_Q.T + (0.0 if b_Q is None else _f64(b_Q)[None, :])
    K, V = hidden_request_kv(X, W_KV, b_KV)
    Hk = n_heads * K.shape[1] // d                # GQA (R18): K/V heads
    Q = rope(Q, np.arange(L), rope_theta, n_heads)
    K = rope(K, np.arange(L), rope_theta, Hk)
    Y = np.empty((L, d))
    for i in range(L):
        o, _ = attend(Q[i], K[: i + 1], V[: i + 1], n_heads, scale, n_kv_heads=Hk)
        Y[i] = W_O @ o + (0.0 if b_O is None else _f64(b_O))
    return Y, K, V


def max_rel_err(gpu, ref, n_heads: int) -> float:
    """Normwise error per (request, head) row (reading R12):
    max_{i,h,c} |gpu - ref| / max(max_c' |ref_{i,h,c'}|, 1e-6)."""
    g = _f64(gpu)
    r = _f64(ref)
    g = g.reshape(g.shape[0], n_heads, -1)
    r = r.reshape(r.shape[0], n_heads, -1)
    denom = np.maximum(np.abs(r).max(axis=2, keepdims=True), 1e-6)
    return float((np.abs(g - r) / denom).max()) if g.size else 0.0
