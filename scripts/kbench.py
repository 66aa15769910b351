#!/usr/bin/env python
"""Per-kernel timing of the scan on synthetic inputs (development aid; the
reported numbers come from bench.py).  Usage: python scripts/kbench.py [c4|c1|c2|c3] ..."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api  # noqa: E402

IMPL = os.environ.get("BPPSA_LEAF_IMPL", "auto")
CFG = {"c4": (1 << 20, 16, 64, 128, 32), "c1": (1000, 16, 20, 8, 8), "c2": (30000, 16, 20, 16, 16),
       "c4s": (1 << 18, 16, 64, 128, 32), "c4b128": (1 << 20, 16, 64, 128, 32), "c4b128c64": (1 << 20, 16, 64, 128, 64),
       "c4c64": (1 << 20, 16, 64, 64, 64), "c4b256": (1 << 20, 16, 64, 256, 32), "c4b512": (1 << 20, 16, 64, 512, 32),
       "c4b256c64": (1 << 20, 16, 64, 256, 64), "c4b512c16": (1 << 20, 16, 64, 512, 16),
       "c4b512c64": (1 << 20, 16, 64, 512, 64), "c4b384": (1 << 20, 16, 64, 384, 32),
       "c4b1024": (1 << 20, 16, 64, 1024, 32), "c4b1024c16": (1 << 20, 16, 64, 1024, 16),
       "c4b768": (1 << 20, 16, 64, 768, 32), "c4sb1024": (1 << 18, 16, 64, 1024, 32),
       "c4b512c28": (1 << 20, 16, 64, 512, 28), "c4b512c24": (1 << 20, 16, 64, 512, 24),
       "c4b448c32": (1 << 20, 16, 64, 448, 32), "c4b1024c8": (1 << 20, 16, 64, 1024, 8),
       "c4b1024c64": (1 << 20, 16, 64, 1024, 64), "c2b8": (30000, 16, 20, 8, 8), "c2b32": (30000, 16, 20, 32, 16),
       "c2b64": (30000, 16, 20, 64, 16), "c2b32c32": (30000, 16, 20, 32, 32), "c2b16c8": (30000, 16, 20, 16, 8),
       "c4b886": (1 << 20, 16, 64, 886, 32), "c4b880": (1 << 20, 16, 64, 880, 32), "c4b947": (1 << 20, 16, 64, 947, 32),
       "c4b840": (1 << 20, 16, 64, 840, 32)}


def run(name, reps=5):
    T, B, H, C0, C = CFG[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    h = (torch.rand((T, B, H), device="cuda", generator=g) * 1.6 - 0.8)
    W = (torch.rand((H, H), device="cuda", generator=g) * 2 - 1) / H ** 0.5
    seed = torch.randn((B, H), device="cuda", generator=g)
    x = (torch.rand((T, B, 1), device="cuda", generator=g) < 0.5).float()
    jac = api.jacobians_rnn(h, W)
    grad = torch.empty_like(h)
    ws = api.workspace(api.scan_workspace_size(jac, "blocked", C0, C))
    wsw = api.workspace(api.weight_grads_workspace_size(T, B, H, 1))
    for _ in range(2):
        api.scan(jac, seed, grad_h=grad, ws=ws, block0=C0, block=C, leaf_impl=IMPL)
    torch.cuda.synchronize()
    traces = [api.LaunchTrace(32) for _ in range(reps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in traces:
        api.scan(jac, seed, grad_h=grad, ws=ws, block0=C0, block=C, trace=t, leaf_impl=IMPL)
    e1.record()
    torch.cuda.synchronize()
    tot = e0.elapsed_time(e1) / reps
    ks = [statistics.median(t.kernel_ms(i) for t in traces) for i in range(traces[0].launches)]
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    api.weight_grads_rnn(x, h, grad, ws=wsw)
    w0.record()
    for _ in range(reps):
        api.weight_grads_rnn(x, h, grad, ws=wsw)
    w1.record()
    torch.cuda.synchronize()
    flops0 = B * T * 2.0 * H ** 3
    print(f"{name} [{IMPL}]: scan {tot:.3f} ms  kernels {[round(k, 3) for k in ks]}  wgrad {w0.elapsed_time(w1) / reps:.3f} ms"
          f"  leaf_up {flops0 / ks[0] / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c4"]:
        run(n)
