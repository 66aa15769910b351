"""Hash of bppsa_scan outputs at H = 20 / 32 (C1, C2 shapes; dev aid: run under two
builds to check that a kernel change is bit-identical)."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api  # noqa: E402

out = []
for T, B, H, C0, C in [(1000, 16, 20, 8, 8), (30000, 16, 20, 16, 16), (3001, 5, 17, 16, 8), (4096, 3, 32, 64, 16)]:
    g = torch.Generator(device="cuda").manual_seed(T + H)
    h = torch.rand((T, B, H), device="cuda", generator=g) * 1.6 - 0.8
    W = (torch.rand((H, H), device="cuda", generator=g) * 2 - 1) / H ** 0.5
    seed = torch.randn((B, H), device="cuda", generator=g)
    jac = api.jacobians_rnn(h, W)
    grad, gi = api.scan(jac, seed, grad_h_init=True, block0=C0, block=C)
    torch.cuda.synchronize()
    dig = hashlib.sha1(grad.cpu().numpy().tobytes() + gi.cpu().numpy().tobytes()).hexdigest()[:16]
    out.append(f"T{T}H{H}:{dig}")
print(" ".join(out))
