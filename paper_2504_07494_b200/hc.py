"""Thin ctypes binding of libhc.so (include/hc.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only turns
torch tensors into pointers and status codes into exceptions.  There is no fallback: if
libhc.so is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# HC_LIB_VARIANT=diag loads the diagnostic build (build.py --diag: timing modes, timeline
# stamps) for experiments; the default is the shipped library.
LIB_PATH = os.path.join(_HERE, "libhc_diag.so" if os.environ.get("HC_LIB_VARIANT") == "diag" else "libhc.so")
# HC_LIB_FILE=<name>.so (same directory): another build of the library, for same-box A/B runs of
# two code versions (scripts/env_ab.sh)
if os.environ.get("HC_LIB_FILE"):
    LIB_PATH = os.path.join(_HERE, os.path.basename(os.environ["HC_LIB_FILE"]))

HC_OK, HC_E_INVALID, HC_E_OOM, HC_E_UNKNOWN_REQ, HC_E_MODE_MISMATCH, HC_E_CUDA, HC_E_UNSUPPORTED, \
    HC_E_WORKSPACE = range(8)
STATUS_NAMES = {0: "HC_OK", 1: "HC_E_INVALID", 2: "HC_E_OOM", 3: "HC_E_UNKNOWN_REQ",
                4: "HC_E_MODE_MISMATCH", 5: "HC_E_CUDA", 6: "HC_E_UNSUPPORTED", 7: "HC_E_WORKSPACE"}
HC_MODE_KV, HC_MODE_HIDDEN = 0, 1
HC_BF16, HC_F32 = 0, 1
HC_FLAG_ACCOUNTING_ONLY, HC_FLAG_FORCE_SIMT, HC_FLAG_GENERIC_ATTN, HC_FLAG_ABSORB_HIDDEN = 1, 2, 4, 8


class HcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class PoolConfig(ctypes.Structure):
    _fields_ = [
        ("d_model", ctypes.c_int32), ("n_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("block_size", ctypes.c_int32), ("num_blocks", ctypes.c_int64), ("dtype", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("storage", ctypes.c_void_p), ("storage_bytes", ctypes.c_size_t),
        ("w_kv", ctypes.c_void_p), ("b_kv", ctypes.c_void_p), ("device", ctypes.c_int32),
        ("split_tokens", ctypes.c_int32),
        ("w_q", ctypes.c_void_p), ("b_q", ctypes.c_void_p), ("w_o", ctypes.c_void_p), ("b_o", ctypes.c_void_p),
        ("rope_theta", ctypes.c_float),
        ("ln_gamma", ctypes.c_void_p), ("ln_beta", ctypes.c_void_p), ("ln_eps", ctypes.c_float),
        ("n_kv_heads", ctypes.c_int32),
    ]


class SchedConfig(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_double), ("total_units", ctypes.c_double), ("ttft_slo", ctypes.c_double),
                ("tbt_slo", ctypes.c_double), ("fallback", ctypes.c_int32), ("eps", ctypes.c_double),
                ("decay", ctypes.c_double), ("hybrid", ctypes.c_int32), ("block_size", ctypes.c_int32)]


class SchedRequest(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int64), ("running", ctypes.c_int32), ("has_token", ctypes.c_int32),
                ("arrival_time", ctypes.c_double), ("last_token_time", ctypes.c_double),
                ("seq_len", ctypes.c_int64)]


class SchedResult(ctypes.Structure):
    _fields_ = [("iter_type", ctypes.c_int32), ("n_candidates", ctypes.c_int32), ("budget", ctypes.c_double),
                ("objective", ctypes.c_double), ("memory_used", ctypes.c_double)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built (run __graft_entry__.build() or "
                          "python paper_2504_07494_b200/build.py); there is no fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, SZ, VP = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
    pI32, pI64, pF = ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(ctypes.c_float)
    sig = {
        "hc_pool_storage_bytes": (SZ, [ctypes.POINTER(PoolConfig)]),
        "hc_pool_create": (I32, [ctypes.POINTER(PoolConfig), ctypes.POINTER(P)]),
        "hc_pool_destroy": (None, [P]),
        "hc_append": (I32, [P, I32, pI64, pI32, pI32, VP, VP, VP, VP]),
        "hc_free": (I32, [P, I64, pI64]),
        "hc_workspace_size": (SZ, [P, I32, pI64]),
        "hc_decode_attention": (I32, [P, I32, pI64, VP, ctypes.c_float, VP, VP, VP, SZ, VP]),
        "hc_project_append": (I32, [P, I32, pI64, pI32, VP, VP, VP]),
        "hc_output_projection": (I32, [P, I32, VP, VP, VP]),
        "hc_layer_norm": (I32, [P, I32, VP, VP, VP]),
        "hc_merge_partials": (I32, [I32, I32, I32, I32, I32, VP, VP, VP, VP, VP]),
        "hc_layer_workspace_size": (SZ, [P, I32, pI64, pI32]),
        "hc_decode_layer": (I32, [P, I32, pI64, pI32, VP, ctypes.c_float, VP, VP, VP, SZ, VP]),
        "hc_prefill_workspace_size": (SZ, [P, I32, pI32]),
        "hc_prefill_layer": (I32, [P, I32, pI64, pI32, pI32, VP, ctypes.c_float, VP, VP, SZ, VP]),
        "hc_pool_num_free": (I64, [P]),
        "hc_units_needed": (I64, [ctypes.POINTER(PoolConfig), I32, I64]),
        "hc_request_info": (I32, [P, I64, pI32, pI64, pI64]),
        "hc_request_blocks": (I32, [P, I64, I32, pI32, I64, pI64]),
        "hc_last_launch_count": (I32, [P]),
        "hc_last_decode_path": (I32, [P]),
        "hc_last_kernel_config": (I32, [P]),
        "hc_set_profiling": (I32, [P, I32]),
        "hc_kernel_times": (I32, [P, pF, pI32]),
        "hc_schedule": (I32, [ctypes.POINTER(SchedConfig), I32, ctypes.POINTER(SchedRequest), ctypes.c_double,
                              pI32, pI32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(SchedResult)]),
        "hc_calibrate_rho": (ctypes.c_double, [I32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
        "hc_last_error": (ctypes.c_char_p, []),
        "hc_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def _check(status: int):
    if status != HC_OK:
        raise HcError(status, lib.hc_last_error().decode())


def _i64(vals: Sequence[int]):
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])


def _i32(vals: Sequence[int]):
    return (ctypes.c_int32 * len(vals))(*[int(v) for v in vals])


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


# ------------------------------------------------------------------ raw C-ABI mirrors
def hc_pool_storage_bytes(cfg: PoolConfig) -> int:
    return int(lib.hc_pool_storage_bytes(ctypes.byref(cfg)))


def hc_units_needed(cfg: PoolConfig, mode: int, n_tokens: int) -> int:
    u = int(lib.hc_units_needed(ctypes.byref(cfg), int(mode), int(n_tokens)))
    if u < 0:
        raise HcError(HC_E_INVALID, lib.hc_last_error().decode())
    return u


def units_needed(d_model: int, n_heads: int, head_dim: int, block_size: int, mode: int, n_tokens: int,
                 dtype: int = HC_BF16, n_kv_heads: int = 0) -> int:
    """Unit blocks of one request (the library's allocation rule; for sizing pools)."""
    cfg = PoolConfig(d_model, n_heads, head_dim, block_size, 1, dtype, HC_FLAG_ACCOUNTING_ONLY)
    cfg.n_kv_heads = int(n_kv_heads)
    return hc_units_needed(cfg, mode, n_tokens)


def hc_pool_create(cfg: PoolConfig) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(lib.hc_pool_create(ctypes.byref(cfg), ctypes.byref(h)))
    return h


def hc_pool_destroy(h) -> None:
    lib.hc_pool_destroy(h)


def hc_append(h, req_ids, modes, n_tokens, k=None, v=None, x=None, stream=None) -> None:
    n = len(req_ids)
    s = _stream(stream) if (k is not None or x is not None) else ctypes.c_void_p(None)
    _check(lib.hc_append(h, n, _i64(req_ids), _i32(modes), _i32(n_tokens), _ptr(k), _ptr(v), _ptr(x), s))


def hc_free(h, req_id: int) -> int:
    rel = ctypes.c_int64(0)
    _check(lib.hc_free(h, int(req_id), ctypes.byref(rel)))
    return rel.value


def hc_workspace_size(h, req_ids) -> int:
    n = int(lib.hc_workspace_size(h, len(req_ids), _i64(req_ids)))
    if n == 0 and len(req_ids) > 0:
        raise HcError(HC_E_INVALID, lib.hc_last_error().decode())
    return n


def hc_decode_attention(h, req_ids, q, scale, out, lse, workspace, stream=None) -> None:
    _check(lib.hc_decode_attention(h, len(req_ids), _i64(req_ids), _ptr(q), float(scale), _ptr(out), _ptr(lse),
                                   _ptr(workspace), workspace.numel() * workspace.element_size()
                                   if workspace is not None else 0, _stream(stream)))


def hc_project_append(h, req_ids, modes, x, q_out, stream=None) -> None:
    _check(lib.hc_project_append(h, len(req_ids), _i64(req_ids), _i32(modes), _ptr(x), _ptr(q_out), _stream(stream)))


def hc_layer_norm(h, n_rows, x, u, stream=None) -> None:
    _check(lib.hc_layer_norm(h, int(n_rows), _ptr(x), _ptr(u), _stream(stream)))


def hc_merge_partials(outs, lses, out, lse=None, stream=None) -> None:
    """outs [P, rows, H*dh] (bf16/fp32), lses [P, rows, H] fp32 -> out [rows, H*dh], lse [rows, H]."""
    if lses.dim() != 3 or outs.dim() != 3:
        raise ValueError("merge: outs [P, rows, H*dh] and lses [P, rows, H] expected")
    n_parts, n_rows, n_heads = lses.shape
    if outs.dtype not in (torch.bfloat16, torch.float32) or out.dtype != outs.dtype:
        raise ValueError(f"merge: outs/out must share dtype bf16 or fp32 (got {outs.dtype}, {out.dtype})")
    if lses.dtype != torch.float32 or (lse is not None and lse.dtype != torch.float32):
        raise ValueError("merge: lses / lse must be fp32")
    hd = outs.shape[2]
    if outs.shape[:2] != (n_parts, n_rows) or hd % n_heads != 0 or tuple(out.shape) != (n_rows, hd) or \
            (lse is not None and tuple(lse.shape) != (n_rows, n_heads)):
        raise ValueError("merge: shapes must be outs [P,rows,H*dh], lses [P,rows,H], out [rows,H*dh], lse [rows,H]")
    for t in (outs, lses, out) + ((lse,) if lse is not None else ()):
        if not (t.is_cuda and t.is_contiguous()):
            raise ValueError("merge: every tensor must be a contiguous CUDA tensor")
    dt = HC_F32 if outs.dtype == torch.float32 else HC_BF16
    _check(lib.hc_merge_partials(int(n_parts), int(n_rows), int(n_heads), int(outs.shape[2] // n_heads), dt,
                                 _ptr(outs), _ptr(lses), _ptr(out), _ptr(lse), _stream(stream)))


def hc_output_projection(h, n_req, o, y, stream=None) -> None:
    _check(lib.hc_output_projection(h, int(n_req), _ptr(o), _ptr(y), _stream(stream)))


def hc_layer_workspace_size(h, req_ids, modes) -> int:
    n = int(lib.hc_layer_workspace_size(h, len(req_ids), _i64(req_ids), _i32(modes)))
    if n == 0 and len(req_ids) > 0:
        raise HcError(HC_E_INVALID, lib.hc_last_error().decode())
    return n


def hc_decode_layer(h, req_ids, modes, x, scale, y, lse, workspace, stream=None) -> None:
    _check(lib.hc_decode_layer(h, len(req_ids), _i64(req_ids), _i32(modes), _ptr(x), float(scale), _ptr(y),
                               _ptr(lse), _ptr(workspace), workspace.numel() * workspace.element_size(),
                               _stream(stream)))


def schedule(cfg: dict, reqs, now: float):
    """hc_schedule: returns (alpha, beta, g, result-dict) for dict-described requests
    (keys of SchedRequest) under dict cfg (keys of SchedConfig)."""
    n = len(reqs)
    c = SchedConfig(*[cfg[k] for k, _ in SchedConfig._fields_])
    arr = (SchedRequest * max(1, n))(*[SchedRequest(*[r[k] for k, _ in SchedRequest._fields_]) for r in reqs])
    a, b = (ctypes.c_int32 * max(1, n))(), (ctypes.c_int32 * max(1, n))()
    g = (ctypes.c_double * max(1, n))()
    res = SchedResult()
    _check(lib.hc_schedule(ctypes.byref(c), n, arr, float(now), a, b, g, ctypes.byref(res)))
    return list(a[:n]), list(b[:n]), list(g[:n]), {k: getattr(res, k) for k, _ in SchedResult._fields_}


def calibrate_rho(m, t) -> float:
    n = len(m)
    r = lib.hc_calibrate_rho(n, (ctypes.c_double * max(1, n))(*m), (ctypes.c_double * max(1, n))(*t))
    if r < 0:
        raise HcError(HC_E_INVALID, "degenerate calibration samples")
    return r


# ------------------------------------------------------------------ convenience owner
_TORCH_DT = {HC_BF16: torch.bfloat16, HC_F32: torch.float32}


class HybridCachePool:
    """Owns the torch storage of one pool and marshals calls to libhc.so."""

    def __init__(self, d_model: int, n_heads: int, head_dim: int, block_size: int, num_blocks: int,
                 dtype: int, w_kv: Optional[torch.Tensor] = None, b_kv: Optional[torch.Tensor] = None,
                 device: int = 0, flags: int = 0, split_tokens: int = 0,
                 w_q: Optional[torch.Tensor] = None, b_q: Optional[torch.Tensor] = None,
                 w_o: Optional[torch.Tensor] = None, b_o: Optional[torch.Tensor] = None,
                 rope_theta: float = 0.0, ln_gamma: Optional[torch.Tensor] = None,
                 ln_beta: Optional[torch.Tensor] = None, ln_eps: float = 1e-5, n_kv_heads: int = 0):
        self.cfg = PoolConfig(d_model, n_heads, head_dim, block_size, num_blocks, dtype, flags, None, 0,
                              None, None, device, split_tokens)
        self.cfg.rope_theta = float(rope_theta)
        self.cfg.ln_eps = float(ln_eps)
        self.cfg.n_kv_heads = int(n_kv_heads)
        self.Hk = int(n_kv_heads) or n_heads
        self.dk = self.Hk * head_dim
        self.dtype = dtype
        self.tdtype = _TORCH_DT[dtype]
        self.d, self.H, self.dh, self.B = d_model, n_heads, head_dim, block_size
        self.device = device
        self.storage = None
        if not flags & HC_FLAG_ACCOUNTING_ONLY:
            # optional projection weights first: the storage layout depends on them
            self._keep = []
            for name, t, shape, dt in (("w_q", w_q, (d_model, d_model), self.tdtype),
                                       ("b_q", b_q, (d_model,), torch.float32),
                                       ("w_o", w_o, (d_model, d_model), self.tdtype),
                                       ("b_o", b_o, (d_model,), torch.float32),
                                       ("ln_gamma", ln_gamma, (d_model,), torch.float32),
                                       ("ln_beta", ln_beta, (d_model,), torch.float32)):
                if t is None:
                    continue
                assert t.is_cuda and t.dtype == dt and tuple(t.shape) == shape, name
                t = t.contiguous()
                self._keep.append(t)
                setattr(self.cfg, name, t.data_ptr())
            nbytes = hc_pool_storage_bytes(self.cfg)
            if nbytes == 0:
                raise HcError(HC_E_INVALID, lib.hc_last_error().decode())
            dev = torch.device("cuda", device)
            self.storage = torch.empty(nbytes + 1024, dtype=torch.uint8, device=dev)
            base = self.storage.data_ptr()
            off = (-base) % 1024
            self.cfg.storage = base + off
            self.cfg.storage_bytes = nbytes
            assert w_kv is not None and w_kv.is_cuda and w_kv.dtype == self.tdtype and w_kv.is_contiguous()
            assert tuple(w_kv.shape) == (2 * self.dk, d_model)
            self.cfg.w_kv = w_kv.data_ptr()
            if b_kv is not None:
                assert b_kv.is_cuda and b_kv.dtype == torch.float32 and b_kv.numel() == 2 * self.dk
                self._b_keep = b_kv.contiguous()
                self.cfg.b_kv = self._b_keep.data_ptr()

        self.handle = hc_pool_create(self.cfg)
        self._ws = None

    def close(self):
        if getattr(self, "handle", None) and hc_pool_destroy is not None:   # None at interpreter exit
            hc_pool_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()

    # -- cache management
    def append(self, req_ids, modes, n_tokens, k=None, v=None, x=None, stream=None):
        for t in (k, v, x):
            if t is not None:
                assert t.is_cuda and t.dtype == self.tdtype and t.is_contiguous(), "rows must be contiguous device tensors"
        hc_append(self.handle, req_ids, modes, n_tokens, k, v, x, stream)

    def free(self, req_id) -> int:
        return hc_free(self.handle, req_id)

    def num_free(self) -> int:
        return int(lib.hc_pool_num_free(self.handle))

    def request_info(self, req_id):
        m, n, u = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib.hc_request_info(self.handle, int(req_id), ctypes.byref(m), ctypes.byref(n), ctypes.byref(u)))
        return m.value, n.value, u.value

    def request_blocks(self, req_id, kind=0):
        cnt = ctypes.c_int64()
        _check(lib.hc_request_blocks(self.handle, int(req_id), kind, None, 0, ctypes.byref(cnt)))
        buf = (ctypes.c_int32 * max(1, cnt.value))()
        _check(lib.hc_request_blocks(self.handle, int(req_id), kind, buf, cnt.value, ctypes.byref(cnt)))
        return list(buf[:cnt.value])

    # -- decode
    def workspace_size(self, req_ids) -> int:
        return hc_workspace_size(self.handle, req_ids)

    def workspace(self, req_ids) -> torch.Tensor:
        n = self.workspace_size(req_ids)
        if self._ws is None or self._ws.numel() < n:
            self._ws = torch.empty(n, dtype=torch.uint8, device=torch.device("cuda", self.device))
        return self._ws

    def decode(self, req_ids, q, scale, out=None, lse=None, want_lse=True, workspace=None, stream=None):
        n = len(req_ids)
        assert q.is_cuda and q.dtype == self.tdtype and q.is_contiguous() and tuple(q.shape) == (n, self.d)
        if out is None:
            out = torch.empty((n, self.d), dtype=self.tdtype, device=q.device)
        if lse is None and want_lse:
            lse = torch.empty((n, self.H), dtype=torch.float32, device=q.device)
        ws = workspace if workspace is not None else self.workspace(req_ids)
        hc_decode_attention(self.handle, req_ids, q, scale, out, lse, ws, stream)
        return out, lse

    # -- the rest of the attention module (f1)
    def project_append(self, req_ids, modes, x, q_out=None, stream=None):
        assert x.is_cuda and x.dtype == self.tdtype and x.is_contiguous() and tuple(x.shape) == (len(req_ids), self.d)
        if q_out is None:
            q_out = torch.empty_like(x)
        hc_project_append(self.handle, req_ids, modes, x, q_out, stream)
        return q_out

    def layer_norm(self, x, u=None, stream=None):
        """u = LN(x) with the pool's pre-attention LayerNorm (hc_layer_norm)."""
        if u is None:
            u = torch.empty_like(x)
        hc_layer_norm(self.handle, x.shape[0], x, u, stream)
        return u

    def output_projection(self, o, y=None, stream=None):
        assert o.is_cuda and o.dtype == self.tdtype and o.is_contiguous() and o.shape[1] == self.d
        if y is None:
            y = torch.empty_like(o)
        hc_output_projection(self.handle, o.shape[0], o, y, stream)
        return y

    def decode_layer(self, req_ids, modes, x, scale, y=None, want_lse=True, stream=None):
        n = len(req_ids)
        assert x.is_cuda and x.dtype == self.tdtype and x.is_contiguous() and tuple(x.shape) == (n, self.d)
        if y is None:
            y = torch.empty_like(x)
        lse = torch.empty((n, self.H), dtype=torch.float32, device=x.device) if want_lse else None
        ws = torch.empty(hc_layer_workspace_size(self.handle, req_ids, modes), dtype=torch.uint8, device=x.device)
        hc_decode_layer(self.handle, req_ids, modes, x, scale, y, lse, ws, stream)
        return y, lse

    def prefill_layer(self, req_ids, modes, lens, x, scale, y=None, stream=None):
        """Prefill / recompute of new requests: x [sum lens, d] -> y [sum lens, d]; caches filled."""
        rows = int(sum(lens))
        assert x.is_cuda and x.dtype == self.tdtype and x.is_contiguous() and tuple(x.shape) == (rows, self.d)
        if y is None:
            y = torch.empty_like(x)
        n = int(lib.hc_prefill_workspace_size(self.handle, len(lens), _i32(lens)))
        if n == 0:
            raise HcError(HC_E_INVALID, lib.hc_last_error().decode())
        ws = torch.empty(n, dtype=torch.uint8, device=x.device)
        _check(lib.hc_prefill_layer(self.handle, len(req_ids), _i64(req_ids), _i32(modes), _i32(lens), _ptr(x),
                                    float(scale), _ptr(y), _ptr(ws), n, _stream(stream)))
        return y

    # -- measurement hooks
    def last_launch_count(self) -> int:
        return int(lib.hc_last_launch_count(self.handle))

    def last_kernel_config(self) -> int:
        return int(lib.hc_last_kernel_config(self.handle))

    def last_decode_path(self) -> int:
        return int(lib.hc_last_decode_path(self.handle))

    def set_profiling(self, on: bool):
        _check(lib.hc_set_profiling(self.handle, 1 if on else 0))

    def kernel_times(self):
        ms = (ctypes.c_float * 4)()
        n = ctypes.c_int32()
        _check(lib.hc_kernel_times(self.handle, ms, ctypes.byref(n)))
        return {"recon_ms": ms[0], "attn_ms": ms[1], "combine_ms": ms[2], "upload_ms": ms[3], "calls": n.value}
