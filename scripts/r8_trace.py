"""Dev aid: per-phase clock64 trace of the ring fold (tc_fold_i8r_kernel) on
CTA 0, each tile group's warp 0.  Build with BPPSA_NVCC_EXTRA=-DBPPSA_F8_TRACE
(force); run: python scripts/r8_trace.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api  # noqa: E402

T, B, H = 1 << 16, 16, 64
g = torch.Generator(device="cuda").manual_seed(0)
h = (torch.rand((T, B, H), device="cuda", generator=g) * 1.6 - 0.8)
W = (torch.rand((H, H), device="cuda", generator=g) * 2 - 1) / H ** 0.5
seed = torch.randn((B, H), device="cuda", generator=g)
jac = api.jacobians_rnn(h, W)
for _ in range(2):
    api.scan(jac, seed, block0=1024, block=32, leaf_impl="int8")
torch.cuda.synchronize()
buf = np.zeros((32, 4096), dtype=np.int64)
api._lib.bppsa_debug_r8_trace(buf.ctypes.data_as(ctypes.c_void_p))
lo, hi = 300, 900
names = ["D wait", "read-out (regions -> y)", "max + digits", "group barrier", "accumulator wait"]
for gr in range(4):
    d = buf[gr * 8:(gr + 1) * 8]
    print(f"group {gr}: median cycles, steps {lo}..{hi}")
    for i, nm in enumerate(names):
        print(f"  {nm:26s} {np.median(d[i + 1, lo:hi] - d[i, lo:hi]):8.0f}")
    print(f"  {'issue -> D ready':26s} {np.median(d[1, lo + 1:hi + 1] - d[5, lo:hi]):8.0f}")
    print(f"  {'step period':26s} {np.median(np.diff(d[5, lo:hi])):8.0f}")
# all MMA batches on CTA 0 in issue order: gaps between consecutive issues
iss = np.sort(np.concatenate([buf[gr * 8 + 5, lo:hi] for gr in range(4)]))
gaps = np.diff(iss)
print("issue-to-issue over all groups: median", np.median(gaps), "mean", gaps.mean(),
      "p10/p90", np.percentile(gaps, 10), np.percentile(gaps, 90))
tick = np.concatenate([buf[gr * 8 + 6, lo:hi] for gr in range(4)])
print("tickets in range:", tick.min(), tick.max())
