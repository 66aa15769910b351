"""Sequential BP on the GPU (bppsa_scan mode LINEAR) at C4 shapes, T = 2^17
(dev aid; bench.py reports the full-T number)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api  # noqa: E402

for H in (64, 20):
    T, B = 1 << 17, 16
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.rand((T, B, H), device="cuda", generator=g) * 1.6 - 0.8
    W = (torch.rand((H, H), device="cuda", generator=g) * 2 - 1) / H ** 0.5
    seed = torch.randn((B, H), device="cuda", generator=g)
    jac = api.jacobians_rnn(h, W)
    grad = torch.empty_like(h)
    ws = api.workspace(api.scan_workspace_size(jac, "linear"))
    api.scan(jac, seed, grad_h=grad, ws=ws, mode="linear")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    api.scan(jac, seed, grad_h=grad, ws=ws, mode="linear")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H={H} T=2^17 linear {ms:.2f} ms = {ms * 1e6 / T:.0f} ns/step; x8 -> T=2^20 {ms * 8:.1f} ms")
