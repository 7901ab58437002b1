"""Seeded synthetic workloads for the five BASELINE.json configs.

Structure (context lengths, cache modes) comes from numpy's PCG64 `default_rng(seed)`
(platform-independent); tensor values come from `synth.rng` (counter-based, identical
on CPU and CUDA).  Nothing here computes any part of the method.

Recipe (DESIGN.md §"Input recipe"):
* tiny   — d=32, H=2x16, B=16, n=[64,1,33,16], modes [KV,KV,hidden,hidden], fp32.
* cfg2   — OPT-13B layer shape (d=5120, 40x128), 64 requests, ShareGPT-like snapshot,
           50% hidden by seeded permutation, bf16.
* cfg3   — OPT-30B layer shape (d=7168, 56x128), 128 candidates, ShareGPT-like, beta from
           the native greedy planner (hc_schedule, via synth.planner), bf16.
* cfg4   — OPT-66B layer shape (d=9216, 72x128), 256 requests, long contexts
           n = clip(round(exp(N(ln 1024, 0.75))), 32, 4096), 50% hidden, bf16.
* cfg5   — cfg4 contexts with hidden fraction h in {0,1/64,...,1} as nested prefixes of
           one seeded permutation.
Tensor values: X ~ N(0,1); W_K, W_V ~ N(0, 1/d); KV-mode K, V ~ N(0,1); q ~ N(0,1);
bias off by default, N(0, 0.02^2) when enabled.  (Irwin-Hall-4 approximations, see rng.)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import rng

MODE_KV = 0
MODE_HIDDEN = 1


@dataclass(frozen=True)
class LayerShape:
    name: str
    d: int
    H: int
    dh: int
    Hk: int = 0    # key/value heads (GQA, the §6.6 models); 0 = H (multi-head)

    @property
    def n_kv(self) -> int:
        return self.Hk or self.H

    @property
    def dk(self) -> int:
        """Width of one K (or V) row: Hk * dh (= d for multi-head attention)."""
        return self.n_kv * self.dh


TINY = LayerShape("tiny", 32, 2, 16)
OPT13B = LayerShape("OPT-13B", 5120, 40, 128)
OPT30B = LayerShape("OPT-30B", 7168, 56, 128)
OPT66B = LayerShape("OPT-66B", 9216, 72, 128)
# §6.6 long-context GQA models: 32 query heads over 8 (LLaMA-3-8B) / 4 (Yi-6B) K/V heads
LLAMA3_8B = LayerShape("LLaMA3-8B", 4096, 32, 128, 8)
YI_6B = LayerShape("Yi-6B", 4096, 32, 128, 4)


@dataclass
class Workload:
    name: str
    shape: LayerShape
    block_size: int
    dtype: str                 # "bf16" | "f32"
    seed: int
    n: List[int]               # context length incl. the current token (n_i >= 1)
    modes: List[int]           # beta_i: 0 = KV cache, 1 = hidden cache
    req_ids: List[int]
    bias: bool = False
    q_scale: float = 1.0       # 4.0 = "peaky" variant
    note: str = ""

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.shape.dh)

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    def n_tokens(self, mode: Optional[int] = None) -> int:
        return int(sum(n for n, m in zip(self.n, self.modes) if mode is None or m == mode))

    def subset(self, idx: List[int], name: str = None) -> "Workload":
        return Workload(name or (self.name + "-subset"), self.shape, self.block_size, self.dtype,
                        self.seed, [self.n[i] for i in idx], [self.modes[i] for i in idx],
                        [self.req_ids[i] for i in idx], self.bias, self.q_scale, self.note)

    # ---- tensors (per request; bit-identical on any device) -------------------------
    def q(self, i: int, device="cpu") -> torch.Tensor:
        return rng.normal_tensor(self.seed, rng.STREAM_Q, self.req_ids[i], [self.shape.d],
                                 self.q_scale, self.torch_dtype, device)

    def kv(self, i: int, device="cpu", rows=None):
        """(K, V) of a KV-mode request, [n_i, Dk] each (Dk = Hk*dh); `rows=(a,b)` gives a row range."""
        d = self.shape.dk
        a, b = rows if rows is not None else (0, self.n[i])
        K = rng.normal_tensor(self.seed, rng.STREAM_K, self.req_ids[i], [b - a, d], 1.0,
                              self.torch_dtype, device, offset=a * d)
        V = rng.normal_tensor(self.seed, rng.STREAM_V, self.req_ids[i], [b - a, d], 1.0,
                              self.torch_dtype, device, offset=a * d)
        return K, V

    def x(self, i: int, device="cpu", rows=None) -> torch.Tensor:
        """Cached input hidden states X of a hidden-mode request, [n_i, d]."""
        d = self.shape.d
        a, b = rows if rows is not None else (0, self.n[i])
        return rng.normal_tensor(self.seed, rng.STREAM_X, self.req_ids[i], [b - a, d], 1.0,
                                 self.torch_dtype, device, offset=a * d)

    def w_kv(self, device="cpu", rows=None) -> torch.Tensor:
        """W_KV = [W_K; W_V], [2 Dk, d] row-major, rows = output features (Eq. 1: k = W_K x)."""
        d = self.shape.d
        a, b = rows if rows is not None else (0, 2 * self.shape.dk)
        out = torch.empty((b - a, d), dtype=self.torch_dtype, device=device)
        step = max(1, (1 << 25) // d)
        for r in range(a, b, step):
            e = min(b, r + step)
            out[r - a:e - a] = rng.normal_tensor(self.seed, rng.STREAM_W, 0, [e - r, d],
                                                 1.0 / math.sqrt(d), self.torch_dtype, device,
                                                 offset=r * d)
        return out

    def _square(self, stream, device, rows=None):
        d = self.shape.d
        a, b = rows if rows is not None else (0, d)
        return rng.normal_tensor(self.seed, stream, 0, [b - a, d], 1.0 / math.sqrt(d), self.torch_dtype, device,
                                 offset=a * d)

    def w_q(self, device="cpu", rows=None) -> torch.Tensor:
        """W_Q [d, d] (q = W_Q x, Eq. 1), N(0, 1/d)."""
        return self._square(rng.STREAM_WQ, device, rows)

    def w_o(self, device="cpu", rows=None) -> torch.Tensor:
        """W_O [d, d] (output map of Eq. 3), N(0, 1/d)."""
        return self._square(rng.STREAM_WO, device, rows)

    def b_q(self, device="cpu") -> Optional[torch.Tensor]:
        return rng.normal_tensor(self.seed, rng.STREAM_B, 1, [self.shape.d], 0.02, torch.float32, device) \
            if self.bias else None

    def b_o(self, device="cpu") -> Optional[torch.Tensor]:
        return rng.normal_tensor(self.seed, rng.STREAM_B, 2, [self.shape.d], 0.02, torch.float32, device) \
            if self.bias else None

    def ln_gamma(self, device="cpu") -> torch.Tensor:
        """Pre-attention LayerNorm scale [d] fp32: 1 + N(0, 0.1^2) (optional f1 component)."""
        return rng.normal_tensor(self.seed, rng.STREAM_B, 3, [self.shape.d], 0.1, torch.float32, device) + 1.0

    def ln_beta(self, device="cpu") -> torch.Tensor:
        """Pre-attention LayerNorm shift [d] fp32: N(0, 0.02^2)."""
        return rng.normal_tensor(self.seed, rng.STREAM_B, 4, [self.shape.d], 0.02, torch.float32, device)

    def x_t(self, i: int, device="cpu") -> torch.Tensor:
        """Layer input of request i's current token (attention-layer step), N(0,1)."""
        return rng.normal_tensor(self.seed, rng.STREAM_XT, self.req_ids[i], [self.shape.d], 1.0,
                                 self.torch_dtype, device)

    def b_kv(self, device="cpu") -> Optional[torch.Tensor]:
        """Optional bias [2 Dk] (fp32), None when disabled (Eq. 1 has no bias)."""
        if not self.bias:
            return None
        return rng.normal_tensor(self.seed, rng.STREAM_B, 0, [2 * self.shape.dk], 0.02,
                                 torch.float32, device)


# ---- context-length generators ------------------------------------------------------

def sharegpt_like(n_req: int, rs: np.random.Generator) -> List[int]:
    """Length-biased snapshot of a running ShareGPT-like batch:
    P ~ round(exp(N(ln 97.6, 1))), O ~ round(exp(N(ln 205, 1))), both >= 1; reject P+O > 2048
    (OPT position limit); accept with prob O/2048; generated-so-far g ~ U{1..O}; n = P+g."""
    out = []
    while len(out) < n_req:
        P = max(1, int(round(math.exp(rs.normal(math.log(97.6), 1.0)))))
        O = max(1, int(round(math.exp(rs.normal(math.log(205.0), 1.0)))))
        if P + O > 2048:
            continue
        if rs.random() >= O / 2048.0:
            continue
        g = int(rs.integers(1, O + 1))
        out.append(P + g)
    return out


def long_lognormal(n_req: int, rs: np.random.Generator) -> List[int]:
    """n = clip(round(exp(N(ln 1024, 0.75))), 32, 4096)."""
    z = rs.normal(math.log(1024.0), 0.75, size=n_req)
    return [int(min(4096, max(32, round(math.exp(v))))) for v in z]


def _half_hidden(n_req: int, rs: np.random.Generator) -> List[int]:
    perm = rs.permutation(n_req)
    modes = [MODE_KV] * n_req
    for i in perm[: n_req // 2]:
        modes[int(i)] = MODE_HIDDEN
    return modes


# ---- the five configs ----------------------------------------------------------------

def tiny(block_size: int = 16, bias: bool = False) -> Workload:
    return Workload("tiny", TINY, block_size, "f32", 0, [64, 1, 33, 16],
                    [MODE_KV, MODE_KV, MODE_HIDDEN, MODE_HIDDEN], [0, 1, 2, 3], bias,
                    note="4 requests, d=32, 2x16 heads, fp32")


def cfg2(block_size: int = 16) -> Workload:
    rs = np.random.default_rng(1)
    n = sharegpt_like(64, rs)
    return Workload("cfg2-opt13b", OPT13B, block_size, "bf16", 1, n, _half_hidden(64, rs),
                    list(range(64)), note="OPT-13B layer, batch 64, ShareGPT-like, 50% hidden")


def cfg3(block_size: int = 16) -> Workload:
    from .planner import plan_cfg3
    rs = np.random.default_rng(2)
    n_all = sharegpt_like(128, rs)
    alpha, beta = plan_cfg3(n_all, OPT30B, rs)
    idx = [i for i in range(128) if alpha[i]]
    return Workload("cfg3-opt30b", OPT30B, block_size, "bf16", 2, [n_all[i] for i in idx],
                    [beta[i] for i in idx], idx,
                    note="OPT-30B layer, 128 candidates, beta from the greedy planner")


def cfg4(block_size: int = 16, n_req: int = 256, seed: int = 3) -> Workload:
    rs = np.random.default_rng(seed)
    n = long_lognormal(n_req, rs)
    return Workload("cfg4-opt66b", OPT66B, block_size, "bf16", seed, n, _half_hidden(n_req, rs),
                    list(range(n_req)), note="OPT-66B layer, batch 256, long contexts, 50% hidden")


CFG5_FRACTIONS = [0.0, 1 / 64, 1 / 32, 1 / 16, 1 / 8, 1 / 4, 1 / 2, 3 / 4, 1.0]


def cfg5(h: float, block_size: int = 16, n_req: int = 256, seed: int = 3) -> Workload:
    rs = np.random.default_rng(seed)
    n = long_lognormal(n_req, rs)
    perm = np.random.default_rng(seed + 1000).permutation(n_req)
    k = int(round(h * n_req))
    modes = [MODE_KV] * n_req
    for i in perm[:k]:
        modes[int(i)] = MODE_HIDDEN
    return Workload(f"cfg5-opt66b-h{h:.4f}", OPT66B, block_size, "bf16", seed, n, modes,
                    list(range(n_req)), note=f"OPT-66B sweep, hidden fraction {h}")


def gqa(shape: LayerShape = LLAMA3_8B, block_size: int = 16, n_req: int = 256, seed: int = 6) -> Workload:
    """f4 (i): a §6.6 GQA model's layer (LLaMA-3-8B: 32 query / 8 K-V heads), cfg4's
    long-context recipe, 50% hidden.  Hidden tokens cost d = 4096 values, KV tokens 2*Hk*dh =
    2048: under GQA the hidden cache is the LARGER one (DESIGN R18)."""
    rs = np.random.default_rng(seed)
    n = long_lognormal(n_req, rs)
    tag = "llama3-8b" if shape is LLAMA3_8B else shape.name.lower()
    return Workload(f"gqa-{tag}", shape, block_size, "bf16", seed, n, _half_hidden(n_req, rs),
                    list(range(n_req)), note=f"{shape.name} layer (GQA {shape.H}/{shape.n_kv}), batch {n_req}, "
                                             "long contexts, 50% hidden")


def by_name(name: str) -> Workload:
    name = name.lower()
    if name == "tiny":
        return tiny()
    if name in ("cfg2", "opt13b"):
        return cfg2()
    if name in ("cfg3", "opt30b"):
        return cfg3()
    if name in ("cfg4", "opt66b"):
        return cfg4()
    if name.startswith("cfg5:"):
        from fractions import Fraction
        return cfg5(float(Fraction(name.split(":", 1)[1])))   # "cfg5:1/32" or "cfg5:0.03125"
    if name in ("gqa", "llama3-8b", "cfg6"):
        return gqa(LLAMA3_8B)
    if name in ("yi-6b",):
        return gqa(YI_6B)
    raise KeyError(name)


def shard_for_rank(w: Workload, rank: int, world: int) -> Workload:
    """Weak scaling (task rule ⑤): every rank processes its own full batch of the same
    recipe, request ids offset by rank so the tensors differ; no data-path collective."""
    if world == 1:
        return w
    ids = [r + rank * 1_000_003 for r in w.req_ids]
    return Workload(w.name, w.shape, w.block_size, w.dtype, w.seed, list(w.n), list(w.modes),
                    ids, w.bias, w.q_scale, w.note)
