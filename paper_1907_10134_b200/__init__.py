"""paper_1907_10134_b200 — a B200-native BPPSA backward scan (arXiv 1907.10134).

`api` is the ctypes binding of libbppsa.so (include/bppsa.h); `dist` drives
the contiguous-time-shard scan over torch.distributed; `build` compiles the
library for sm_100a.  Importing `api` without the built library raises.
"""
__all__ = ["api", "dist", "build"]
