"""Dev aid: per-phase clock64 trace of the exact-integer fold on CTA 0, both
slots' issuer lanes.  Build with BPPSA_NVCC_EXTRA=-DBPPSA_F8_TRACE (force);
run: python scripts/f8_trace.py"""
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
buf = np.zeros((16, 4096), dtype=np.int64)
api._lib.bppsa_debug_f8_trace(buf.ctypes.data_as(ctypes.c_void_p))
names = ["top (before D wait)", "D ready (bar)", "y computed", "max exchanged", "digits packed", "stored+fenced", "bar passed", "MMAs issued"]
for sl in range(2):
    d = buf[sl * 8:(sl + 1) * 8, 300:1300].astype(np.float64)
    print(f"slot {sl}: median cycles relative to the step's top (steps 300..1300)")
    for i, nm in enumerate(names):
        print(f"  {nm:22s} {np.median(d[i] - d[0]):8.0f}")
    print("  step period:", np.median(np.diff(buf[sl * 8, 300:1300])))
    print("  issue -> D ready (next step):", np.median(buf[sl * 8 + 1, 301:1301] - buf[sl * 8 + 7, 300:1300]))
# cross-slot: when slot 1 issues relative to slot 0's D-ready
print("slot1 issue - slot0 issue (median):", np.median(buf[15, 300:1300] - buf[7, 300:1300]))
