"""Dev aid: per-phase clock64 trace of the exact-integer fold on CTA 0.
Build with BPPSA_NVCC_EXTRA=-DBPPSA_I8_TRACE; run: python scripts/i8_trace.py"""
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
    api.scan(jac, seed, block0=512, block=32, leaf_impl="int8")
torch.cuda.synchronize()
buf = np.zeros((12, 2048), dtype=np.int64)
lib = api._lib
lib.bppsa_debug_i8_trace(buf.ctypes.data_as(ctypes.c_void_p))
names = ["phase start", "D ready", "regions loaded", "pm stored", "exchanged", "arrived", "iss: a ready", "iss: issued",
         "digits packed", "digits stored", "proxy fenced", "-"]
d = buf[:, 200:1200].astype(np.float64)
t0 = d[0]
print("median cycles relative to phase start (phases 200..1200):")
for i, nm in enumerate(names[:11]):
    print(f"  {nm:16s} {np.median(d[i] - t0):8.0f}")
print("phase period:", np.median(np.diff(buf[0, 200:1200])))
print("issue -> D ready (same slot, next step):", np.median(buf[1, 202:1202] - buf[7, 200:1200]))
