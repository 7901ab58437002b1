"""Fused-kernel anatomy from the diagnostic build's per-CTA globaltimer stamps
(build.py --diag; HC_LIB_VARIANT=diag).  Usage: HC_LIB_VARIANT=diag python scripts/timeline.py cfg5:1/32 [...]
Prints, per config: kernel span, when the CTAs' GEMM warps drained (min / median / max),
the share of the KV attention tasks taken by then, and when the attention warps finished."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["HC_LIB_VARIANT"] = "diag"
from paper_2504_07494_b200 import build as hb  # noqa: E402

hb.build(variant="diag")
from paper_2504_07494_b200 import hc  # noqa: E402
from synth import configs as C  # noqa: E402
from synth import drive as D  # noqa: E402

fn = hc.lib.hc_debug_timeline
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
fn.restype = ctypes.c_int
for name in sys.argv[1:]:
    w = C.by_name(name)
    pool = D.make_pool(w)
    D.fill(pool, w)
    q = D.queries(w)
    ids = list(w.req_ids)
    out = torch.empty_like(q)
    ws = pool.workspace(ids)
    spans = []
    for rep in range(int(os.environ.get("REPS", "20"))):
        hc.hc_decode_attention(pool.handle, ids, q, w.scale, out, None, ws)
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (512 * 5))()
        assert fn(buf, 512) == 0
        t = np.frombuffer(buf, dtype=np.uint64).reshape(512, 5)[:torch.cuda.get_device_properties(0).multi_processor_count].astype(np.float64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3   # us
        rel[:, 3] = t[:, 3]    # a task count, not a time
        spans.append(rel)
    rel = np.median(np.stack(spans), axis=0)
    kv_tasks = sum(-(-n // 512) for n, m in zip(w.n, w.modes) if m == 0) * w.shape.H
    res = {"config": name, "diag_attn": os.environ.get("HC_DIAG_ATTN", "0"), "span_us": float(max(rel[:, 2].max(), rel[:, 1].max())),
           "gemm_drain_us": [float(np.min(rel[:, 1])), float(np.median(rel[:, 1])), float(np.max(rel[:, 1]))],
           "attn_first_warp_done_us": [float(np.min(rel[:, 4])), float(np.median(rel[:, 4]))],
           "attn_done_us": [float(np.min(rel[:, 2])), float(np.median(rel[:, 2])), float(np.max(rel[:, 2]))],
           "tasks_taken_at_median_drain": float(np.median(rel[:, 3])), "kv_tasks_total_approx": kv_tasks}
    kvp = int(os.environ.get("HC_KV_PAIRS", "0"))
    if kvp > 0:   # spatial split: CTAs [0, 2G) run the GEMM, the rest only stream KV
        g = rel.shape[0] - 2 * kvp
        res["gemm_ctas_drain_us"] = [float(np.min(rel[:g, 1])), float(np.median(rel[:g, 1])), float(np.max(rel[:g, 1]))]
        res["kv_ctas_attn_done_us"] = [float(np.min(rel[g:, 2])), float(np.median(rel[g:, 2])), float(np.max(rel[g:, 2]))]
        res["gemm_ctas_attn_done_us"] = [float(np.min(rel[:g, 2])), float(np.median(rel[:g, 2])), float(np.max(rel[:g, 2]))]
    print(json.dumps(res), flush=True)
    del pool
