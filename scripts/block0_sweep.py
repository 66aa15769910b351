"""Dev aid: full single-GPU scan time (fold + levels + walk) of a 2^20 / N
time shard of C4 at several level-0 blocks — the per-rank work of bench.py
at N ranks (the exchange adds ~tens of us).  python scripts/block0_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api  # noqa: E402

B, H = 16, 64
for N in (1, 2, 4, 8):
    T = (1 << 20) // N
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.rand((T, B, H), device="cuda", generator=g) * 1.6 - 0.8
    W = (torch.rand((H, H), device="cuda", generator=g) * 2 - 1) / H ** 0.5
    seed = torch.randn((B, H), device="cuda", generator=g)
    jac = api.jacobians_rnn(h, W)
    grad = torch.empty_like(h)
    out = []
    for b0 in (64, 128, 256, 512, 1024, 2048):
        if T // b0 < 8:
            continue
        ws = api.workspace(api.scan_workspace_size(jac, "blocked", b0, 32))
        for _ in range(2):
            api.scan(jac, seed, grad_h=grad, ws=ws, block0=b0, block=32)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            api.scan(jac, seed, grad_h=grad, ws=ws, block0=b0, block=32)
        e1.record()
        torch.cuda.synchronize()
        out.append(f"{b0}: {e0.elapsed_time(e1) / 5:.2f}")
        del ws
    print(f"N={N} (T={T}):", "  ".join(out), flush=True)
    del h, jac, grad
    torch.cuda.empty_cache()
