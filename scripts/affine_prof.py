"""Per-launch times of bppsa_scan_affine at C4 shapes (development aid)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api  # noqa: E402

T, B, H, C0, C = 1 << 20, 16, 64, 512, 32
g = torch.Generator(device="cuda").manual_seed(0)
h = torch.rand((T, B, H), device="cuda", generator=g) * 1.6 - 0.8
W = (torch.rand((H, H), device="cuda", generator=g) * 2 - 1) / H ** 0.5
seed = torch.randn((B, H), device="cuda", generator=g)
e = torch.randn((T, B, H), device="cuda", generator=g) * 0.01
jac = api.jacobians_rnn(h, W)
grad = torch.empty_like(h)
ws = api.workspace(api.scan_workspace_size(jac, "blocked", C0, C))
for fn in ("scan", "scan_affine"):
    f = getattr(api, fn)
    args = (jac, seed, e) if fn == "scan_affine" else (jac, seed)
    for _ in range(2):
        f(*args, grad_h=grad, ws=ws, block0=C0, block=C)
    torch.cuda.synchronize()
    tr = [api.LaunchTrace(32) for _ in range(3)]
    for t in tr:
        f(*args, grad_h=grad, ws=ws, block0=C0, block=C, trace=t)
    torch.cuda.synchronize()
    ks = [round(statistics.median(t.kernel_ms(i) for t in tr), 3) for i in range(tr[0].launches)]
    print(fn, sum(ks), ks)
