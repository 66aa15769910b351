"""Dev aid: per-step clock64 trace of the int8 walk on CTA 0 (build with
BPPSA_NVCC_EXTRA=-DBPPSA_I8_TRACE)."""
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
import ctypes  # noqa: E402
api._lib.bppsa_debug_i8_trace(buf.ctypes.data_as(ctypes.c_void_p))
import os as _os
if _os.environ.get("WT"):      # the TMA walk's events
    names = ["step top", "D+h ready (bar)", "y + v stored", "exchanged", "digits in TMEM", "digit barrier",
             "MMA+TMA issued", "-", "-", "-"]
else:
    names = ["step start", "staged+stored", "h landed", "pm stored", "exchanged", "digits packed", "digits in TMEM",
             "A barrier", "D ready", "regions -> v"]
d = buf[:, 100:500].astype(np.float64)
for i, nm in enumerate(names):
    print(f"  {nm:16s} {np.median(d[i] - d[0]):8.0f}")
print("step period:", np.median(np.diff(buf[0, 100:500])))
