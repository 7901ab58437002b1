"""Stress: repeated decode calls must give bit-identical outputs (catches races in the fused
kernel's cross-CTA tile queue, the split-K task counter and the attend epilogue).
Usage: python scripts/stress_determinism.py [reps] [config ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as C  # noqa: E402
from synth import drive as D  # noqa: E402
from paper_2504_07494_b200 import hc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
names = sys.argv[2:] or ["cfg2", "llama3-8b", "cfg5:1/32", "cfg3"]
bad = 0
for name in names:
    w = C.by_name(name)
    pool = D.make_pool(w)
    D.fill(pool, w)
    q = D.queries(w)
    ids = list(w.req_ids)
    ws = pool.workspace(ids)
    H = w.shape.H
    out0, lse0 = torch.empty_like(q), torch.empty(len(ids), H, dtype=torch.float32, device=q.device)
    hc.hc_decode_attention(pool.handle, ids, q, w.scale, out0, lse0, ws)
    out, lse = torch.empty_like(out0), torch.empty_like(lse0)
    for r in range(reps):
        out.fill_(0)
        hc.hc_decode_attention(pool.handle, ids, q, w.scale, out, lse, ws)
        if not (torch.equal(out, out0) and torch.equal(lse, lse0)):
            bad += 1
            print(name, "rep", r, "MISMATCH", float((out.float() - out0.float()).abs().max()), flush=True)
    torch.cuda.synchronize()
    print(name, "reps", reps, "path", pool.last_decode_path(), "ok" if bad == 0 else f"{bad} mismatches", flush=True)
    del pool
sys.exit(1 if bad else 0)
