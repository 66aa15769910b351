"""C3 (GRU, H = 20, IRMAS L set, B = 64) kernel times for a few block shapes (dev aid)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bppsa_workloads as W  # noqa: E402
from paper_1907_10134_b200 import api  # noqa: E402

gw = W.gru_workload("L", 64, seed=2)
tape = {k: torch.from_numpy(v).cuda() for k, v in gw.tape.items()}
x = torch.from_numpy(gw.x).cuda()
W3, g = torch.from_numpy(gw.params["W_hh3"]).cuda(), torch.from_numpy(gw.g).cuda()
jac = api.jacobians_gru(tape["h_prev"], tape["r"], tape["z"], tape["n"], tape["M"], W3)
grad = torch.empty_like(tape["r"])
ws_w = api.workspace(api.weight_grads_workspace_size(*grad.shape, x.shape[2]))
for b0, b in [(16, 16), (8, 8), (32, 16), (64, 16), (4, 8)]:
    ws = api.workspace(api.scan_workspace_size(jac, "blocked", b0, b))
    for _ in range(3):
        api.scan(jac, g, grad_h=grad, ws=ws, block0=b0, block=b)
    torch.cuda.synchronize()
    trs = [api.LaunchTrace(64) for _ in range(10)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in trs:
        api.scan(jac, g, grad_h=grad, ws=ws, block0=b0, block=b, trace=t)
    e1.record()
    torch.cuda.synchronize()
    ks = [round(statistics.median(t.kernel_ms(i) for t in trs), 4) for i in range(trs[0].launches)]
    print(f"c3 block0 {b0} block {b}: scan {e0.elapsed_time(e1) / 10:.3f} ms kernels {ks}")
w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
api.weight_grads_gru(x, tape, grad, ws=ws_w)
w0.record()
for _ in range(10):
    api.weight_grads_gru(x, tape, grad, ws=ws_w)
w1.record()
torch.cuda.synchronize()
print(f"c3 weight_grads_gru {w0.elapsed_time(w1) / 10:.3f} ms")
