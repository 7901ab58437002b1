"""B200-native hybrid-cache decode attention (Apt-Serve, arXiv 2504.07494, §3.1 / §4.3).

The product is libhc.so (C ABI in include/hc.h, CUDA kernels for sm_100a under csrc/);
`hc` is its thin ctypes binding.  Importing `paper_2504_07494_b200.hc` fails loudly if
the library is not built — there is no CPU or eager-PyTorch fallback.
"""
__all__ = ["hc"]
