"""Crossover anatomy (cfg5, OPT-66B contexts): one pool, decode timed over all requests,
over the hidden-mode requests alone and over the KV-mode requests alone (CUDA events,
same launch path as bench.py).  Prints the fused step time next to the two halves."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_07494_b200 import hc  # noqa: E402
from synth import configs as C  # noqa: E402
from synth import drive as T  # noqa: E402


def time_ids(pool, ids, q, w, steps=int(os.environ.get("CS_STEPS", "20")), warmup=int(os.environ.get("CS_WARMUP", "3"))):
    out = torch.empty((len(ids), w.shape.d), dtype=w.torch_dtype, device="cuda")
    lse = torch.empty((len(ids), w.shape.H), dtype=torch.float32, device="cuda")
    qq = q[[w.req_ids.index(i) for i in ids]].contiguous()
    ws = pool.workspace(ids)
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        hc.hc_decode_attention(pool.handle, ids, qq, w.scale, out, lse, ws, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        hc.hc_decode_attention(pool.handle, ids, qq, w.scale, out, lse, ws, s)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


if __name__ == "__main__":
    torch.cuda.set_device(0)
    hs = [float(x) for x in (sys.argv[1:] or ["0.015625", "0.03125", "0.0625", "0.125"])]
    for h in hs:
        w = C.cfg5(h)
        pool = T.make_pool(w)
        T.fill(pool, w)
        q = T.queries(w)
        hid = [i for i, m in zip(w.req_ids, w.modes) if m == 1]
        kv = [i for i, m in zip(w.req_ids, w.modes) if m == 0]
        r = {"h": h, "all_ms": time_ids(pool, list(w.req_ids), q, w), "hidden_only_ms": time_ids(pool, hid, q, w),
             "kv_only_ms": time_ids(pool, kv, q, w), "n_hidden": len(hid), "n_kv": len(kv)}
        r["sum_ms"] = r["hidden_only_ms"] + r["kv_only_ms"]
        print(json.dumps(r), flush=True)
        del pool
        torch.cuda.empty_cache()
