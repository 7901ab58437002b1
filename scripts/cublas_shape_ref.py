"""Library calibration: cuBLAS (torch.matmul, bf16, fp32 accumulate) on the dense GEMM with
the same M, N, K as the reconstruction of each config (no block gather, no epilogue, no
attention), timed with CUDA events back to back.  Context for the fused kernel's TF/s."""
import json
import sys
import time

import torch

SHAPES = {   # name: (M = hidden rows incl. block padding, from synth.configs; d)
    "cfg2": (13904, 5120),
    "cfg3": (24672, 7168),
    "cfg4": (160240, 9216),
    "cfg5_1/32": (8432, 9216),
}


def run(name, M, d, iters):
    a = torch.randn(M, d, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(2 * d, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5
    for _ in range(3):
        torch.matmul(a, w.t())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        torch.matmul(a, w.t())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 2.0 * M * 2 * d * d
    return {"shape": name, "M": M, "N": 2 * d, "K": d, "ms": ms, "tflops": fl / ms / 1e9}


if __name__ == "__main__":
    out = []
    for name, (M, d) in SHAPES.items():
        iters = max(5, int(2000 / max(1e-3, 2.0 * M * 2 * d * d / 1.3e12)))  # ~2 s of work
        out.append(run(name, M, d, min(iters, 400)))
        print(json.dumps(out[-1]), flush=True)
        time.sleep(2)
    json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cublas_shapes.json", "w"), indent=1)
