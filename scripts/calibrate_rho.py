"""Calibrate the planner's rho on this B200 (Eq. 6, t = rho * m; the paper's ~30 s
pre-serving fit): time the reconstruction GEMM of hidden-only OPT-shaped batches
of increasing total context, regress GEMM time on memory units (KV units of the hidden
tokens) through the origin with hc_calibrate_rho, and print rho per layer."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_07494_b200 import hc
from synth.configs import OPT13B, OPT30B, OPT66B, MODE_HIDDEN, Workload
from tests import hc_testlib as T

out = {}
for shape in (OPT13B, OPT30B, OPT66B):
    ms, ts = [], []
    for n_req, n_tok in ((8, 256), (16, 512), (32, 512), (32, 1024), (64, 1024)):
        w = Workload(f"rho-{shape.name}", shape, 16, "bf16", 9, [n_tok] * n_req, [MODE_HIDDEN] * n_req,
                     list(range(n_req)))
        pool = T.make_pool(w, split_tokens=0)
        T.fill(pool, w)
        q = T.queries(w)
        ws = pool.workspace(w.req_ids)
        os.environ["HC_FUSED"] = "0"   # time the reconstruction GEMM alone
        for _ in range(3):
            pool.decode(w.req_ids, q, w.scale, workspace=ws)
        pool.set_profiling(True)
        pool.kernel_times()
        for _ in range(10):
            pool.decode(w.req_ids, q, w.scale, workspace=ws)
        kt = pool.kernel_times()
        pool.set_profiling(False)
        t = kt["recon_ms"] / kt["calls"] / 1e3
        m = sum(2.0 * (n + 1) for n in w.n)          # KV memory units of the batch (block_size 1)
        ms.append(m)
        ts.append(t)
        pool.close()
        del pool
        torch.cuda.empty_cache()
    rho = hc.calibrate_rho(ms, ts)
    out[shape.name] = {"rho_s_per_unit_per_layer": rho, "samples": list(zip(ms, ts)),
                       "ideal_at_1.4PF": (4.0 * shape.d ** 2 / 1.4e15) / 2.0}
    print(shape.name, f"rho = {rho:.3e} s/unit/layer (ideal at 1.4 PF/s: {out[shape.name]['ideal_at_1.4PF']:.3e})",
          flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/rho_calibration.json", "w"), indent=1)
