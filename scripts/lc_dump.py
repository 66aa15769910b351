"""Dump (or compare against) bppsa_scan outputs at C1 shapes (dev aid for kernel A/B)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api  # noqa: E402

T, B, H, C0, C = 1000, 16, 20, 8, 8
g = torch.Generator(device="cuda").manual_seed(T + H)
h = torch.rand((T, B, H), device="cuda", generator=g) * 1.6 - 0.8
W = (torch.rand((H, H), device="cuda", generator=g) * 2 - 1) / H ** 0.5
seed = torch.randn((B, H), device="cuda", generator=g)
jac = api.jacobians_rnn(h, W)
grad, gi = api.scan(jac, seed, grad_h_init=True, block0=C0, block=C)
out = np.concatenate([grad.cpu().numpy().ravel(), gi.cpu().numpy().ravel()])
if sys.argv[1] == "save":
    np.save("/tmp/lc_ref.npy", out)
else:
    ref = np.load("/tmp/lc_ref.npy")
    d = np.abs(out - ref)
    idx = np.argwhere(d > 0).ravel()
    print("differing", idx.size, "of", out.size, "max abs", d.max(), "max rel", (d / np.maximum(np.abs(ref), 1e-30)).max())
    if idx.size:
        i = idx[0]
        print("first", i, "t,b,h =", np.unravel_index(i, (T, B, H)) if i < T * B * H else "init", out[i], ref[i])
