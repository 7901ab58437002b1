"""Workload driver: builds a libhc pool for a synth.Workload, fills its caches and runs the
decode call — the GPU side of tests and bench.py.  It calls only the product library
(paper_2504_07494_b200.hc) and the seeded input generators; it never imports oracle/
(task rule ③) and holds none of the method's arithmetic (pool sizing asks the library).
"""
from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np
import torch

from synth.configs import MODE_HIDDEN, MODE_KV, Workload


def pool_blocks(w: Workload, slack: float = 0.05) -> int:
    """Unit blocks for the workload's caches + slack (sized by the library's allocation rule)."""
    from paper_2504_07494_b200 import hc
    dt = hc.HC_BF16 if w.dtype == "bf16" else hc.HC_F32
    need = sum(hc.units_needed(w.shape.d, w.shape.H, w.shape.dh, w.block_size, m, n, dt, w.shape.n_kv)
               for n, m in zip(w.n, w.modes))
    return int(need * (1 + slack)) + 4


def _gen(fn, dev, gen: str):
    """Run a synth generator on the device, or on the host (gen="host") and copy the result
    over: the generator is bit-identical on both, and host generation launches no kernels
    (smoke() uses it so the driver's launch capture sees only the library's kernels)."""
    if gen == "host":
        t = fn("cpu")
        if t is None:
            return None
        return tuple(x.to(dev) for x in t) if isinstance(t, tuple) else t.to(dev)
    return fn(dev)


def make_pool(w: Workload, device: int = 0, flags: int = 0, split_tokens: int = 0, num_blocks: int = None,
              w_kv: torch.Tensor = None, b_kv: torch.Tensor = None, rope_theta: float = 0.0, gen: str = "device"):
    from paper_2504_07494_b200 import hc
    dev = torch.device("cuda", device)
    W = w_kv if w_kv is not None else _gen(lambda d: w.w_kv(device=d), dev, gen)
    b = b_kv if b_kv is not None else _gen(lambda d: w.b_kv(device=d), dev, gen)
    dt = hc.HC_BF16 if w.dtype == "bf16" else hc.HC_F32
    return hc.HybridCachePool(w.shape.d, w.shape.H, w.shape.dh, w.block_size,
                              num_blocks or pool_blocks(w), dt, W, b, device, flags, split_tokens,
                              rope_theta=rope_theta, n_kv_heads=w.shape.n_kv)


def fill(pool, w: Workload, device: int = 0, order: str = "rr", data=None, seed: int = 0, gen: str = "device"):
    """Append every request's cache.  order='rr': one block per request per round, so a
    request's blocks are strided across the pool (steady-state server);
    'seq': request by request; 'shuffle': rounds with a seeded request order."""
    dev = torch.device("cuda", device)
    B = w.block_size
    if data is None:
        data = {}
        for i in range(len(w.n)):
            data[i] = _gen((lambda d, i=i: w.kv(i, device=d)) if w.modes[i] == MODE_KV else
                           (lambda d, i=i: w.x(i, device=d)), dev, gen)
    if order == "seq":
        for i in range(len(w.n)):
            _append_rows(pool, w, [i], [(0, w.n[i])], data)
        return data
    rs = np.random.default_rng(seed)
    nrounds = max(math.ceil(n / B) for n in w.n)
    for r in range(nrounds):
        idx = [i for i in range(len(w.n)) if w.n[i] > r * B]
        if order == "shuffle":
            idx = [idx[j] for j in rs.permutation(len(idx))]
        _append_rows(pool, w, idx, [(r * B, min(w.n[i], (r + 1) * B)) for i in idx], data)
    return data


def _append_rows(pool, w, idx, ranges, data):
    ks, vs, xs, toks = [], [], [], []
    for i, (a, b) in zip(idx, ranges):
        toks.append(b - a)
        if w.modes[i] == MODE_KV:
            ks.append(data[i][0][a:b])
            vs.append(data[i][1][a:b])
        else:
            xs.append(data[i][a:b])
    k = torch.cat(ks).contiguous() if ks else None
    v = torch.cat(vs).contiguous() if vs else None
    x = torch.cat(xs).contiguous() if xs else None
    pool.append([w.req_ids[i] for i in idx], [w.modes[i] for i in idx], toks, k, v, x)


def queries(w: Workload, device: int = 0, gen: str = "device") -> torch.Tensor:
    dev = torch.device("cuda", device)
    return _gen(lambda d: torch.stack([w.q(i, device=d) for i in range(len(w.n))]).contiguous(), dev, gen)


def decode(pool, w: Workload, q: torch.Tensor, idx: Optional[Sequence[int]] = None):
    """One decode call; outputs come back to the host before any dtype conversion (no torch
    kernels around the library's)."""
    if idx is None:
        ids, qq = list(w.req_ids), q
    else:
        idx = list(idx)
        ids, qq = [w.req_ids[i] for i in idx], q[idx].contiguous()
    out, lse = pool.decode(ids, qq, w.scale)
    torch.cuda.synchronize()
    return out.cpu().float().numpy(), lse.cpu().numpy()


# ---------------------------------------------------------------- attention layer (f1)
LN_EPS = 1e-5


def make_layer_pool(w: Workload, device: int = 0, num_blocks: int = None, flags: int = 0, rope_theta: float = 0.0,
                    ln: bool = False):
    from paper_2504_07494_b200 import hc
    dev = torch.device("cuda", device)
    dt = hc.HC_BF16 if w.dtype == "bf16" else hc.HC_F32
    lnk = {"ln_gamma": w.ln_gamma(device=dev), "ln_beta": w.ln_beta(device=dev), "ln_eps": LN_EPS} if ln else {}
    return hc.HybridCachePool(w.shape.d, w.shape.H, w.shape.dh, w.block_size, num_blocks or pool_blocks(w),
                              dt, w.w_kv(device=dev), w.b_kv(device=dev), device, flags,
                              w_q=w.w_q(device=dev), b_q=w.b_q(device=dev), w_o=w.w_o(device=dev),
                              b_o=w.b_o(device=dev), rope_theta=rope_theta, n_kv_heads=w.shape.n_kv, **lnk)


def prefix_workload(w: Workload) -> Workload:
    """The same requests with the current token removed (n_i - 1 cached tokens)."""
    return Workload(w.name + "-prefix", w.shape, w.block_size, w.dtype, w.seed, [n - 1 for n in w.n],
                    list(w.modes), list(w.req_ids), w.bias, w.q_scale, w.note)
