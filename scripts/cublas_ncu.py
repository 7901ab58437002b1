"""One cuBLAS bf16 GEMM per shape (for an ncu metrics pass; see scripts/cublas_shape_ref.py)."""
import sys
import torch
for M, d in [(13904, 5120), (160240, 9216)]:
    a = torch.randn(M, d, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(2 * d, d, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        torch.matmul(a, w.t())
    torch.cuda.synchronize()
