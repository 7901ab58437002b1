"""Counter-based seeded tensor generator shared by the bench, the GPU tests and the oracle tests.

This module holds NONE of the method's arithmetic (no projection, no softmax, no
attention).  It only turns (seed, stream, key, element index) into numbers, and it
produces bit-identical results on CPU and on CUDA:

* the hash is 32-bit integer arithmetic done in int64 torch tensors with every
  product kept below 2**63 (16-bit limb multiplication), so it never relies on
  wrap-around;
* the "normal" variate is an Irwin-Hall sum of four 16-bit uniforms: the sum is an
  exact integer (|s| < 2**18, exact in fp32) and is turned into a float by ONE
  correctly rounded fp32 multiply, then rounded (RNE) to the storage dtype.  IEEE
  multiplication and RNE casts give the same bits on every device.

So the oracle side can regenerate any request's inputs on the host, element for
element, without ever reading a tensor back from the CUDA path (task rule ③).
"""
from __future__ import annotations

import math

import torch

_M32 = 0xFFFFFFFF
# stream ids: one per logical tensor family
STREAM_Q = 1
STREAM_K = 2
STREAM_V = 3
STREAM_X = 4
STREAM_W = 5
STREAM_B = 6
STREAM_WQ = 7
STREAM_WO = 8
STREAM_XT = 9   # layer input of the current (new) token

_IH4_STD = 65536.0 / math.sqrt(3.0)  # std of (k1+k2+k3+k4) for k_i ~ U{0..65535}
_IH4_MEAN = 4 * 32767.5


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2**32 for 0 <= x, c < 2**32 without int64 overflow."""
    cl, ch = c & 0xFFFF, (c >> 16) & 0xFFFF
    xl = x & 0xFFFF
    xh = x >> 16
    cross = ((xh * cl + xl * ch) & 0xFFFF) << 16
    return (xl * cl + cross) & _M32


def mix32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 integer hash (bijective on 32-bit values)."""
    x = x & _M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _mix_int(v: int) -> int:
    return int(mix32(torch.tensor([v & _M32], dtype=torch.int64))[0])


def stream_key(seed: int, stream: int, key: int) -> int:
    """32-bit base key for one tensor (seed, stream family, per-request / per-layer key)."""
    h = _mix_int(seed * 0x9E3779B1 + 0x632BE5AB)
    h = _mix_int(h ^ (stream * 0x85EBCA77))
    h = _mix_int(h ^ (key & _M32))
    h = _mix_int(h ^ ((key >> 32) & _M32) ^ 0x5BD1E995)
    return h


def normal_tensor(seed: int, stream: int, key: int, shape, std: float,
                  dtype=torch.bfloat16, device="cpu", offset: int = 0) -> torch.Tensor:
    """Approximately N(0, std^2) tensor; element e uses counter (offset + e).

    Bit-identical for the same arguments on any device.  `offset` lets a caller
    generate a row range of a larger logical tensor (e.g. rows [a, b) of X)."""
    numel = 1
    for s in shape:
        numel *= int(s)
    assert offset + numel < 2**31, "counter space exceeded; use another key"
    base = stream_key(seed, stream, key)
    e = torch.arange(offset, offset + numel, dtype=torch.int64, device=device)
    ha = mix32((2 * e) ^ base)
    hb = mix32((2 * e + 1) ^ base)
    s = (ha & 0xFFFF) + (ha >> 16) + (hb & 0xFFFF) + (hb >> 16)
    s = (s - 131070).to(torch.float32)  # exact: |s| <= 131070 < 2**24
    c = torch.tensor(std / _IH4_STD, dtype=torch.float32).item()  # fp32 constant
    z = s * torch.tensor(c, dtype=torch.float32, device=device)
    return z.to(dtype).reshape(tuple(shape))


def uniform_tensor(seed: int, stream: int, key: int, shape, device="cpu") -> torch.Tensor:
    """U[0,1) float64 tensor from the same counter hash (host-side structure use)."""
    numel = 1
    for s in shape:
        numel *= int(s)
    base = stream_key(seed, stream, key)
    e = torch.arange(numel, dtype=torch.int64, device=device)
    h = mix32(e ^ base)
    return (h.to(torch.float64) / 4294967296.0).reshape(tuple(shape))
