"""bppsa_weight_grads_rnn at C4 shapes, 40 reps after warm-up (dev aid)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api  # noqa: E402

T, B, H = 1 << 20, 16, 64
g = torch.Generator(device="cuda").manual_seed(0)
h = torch.rand((T, B, H), device="cuda", generator=g) * 1.6 - 0.8
gr = torch.randn((T, B, H), device="cuda", generator=g)
x = (torch.rand((T, B, 1), device="cuda", generator=g) < 0.5).float()
ws = api.workspace(api.weight_grads_workspace_size(T, B, H, 1))
for _ in range(5):
    api.weight_grads_rnn(x, h, gr, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(40):
    api.weight_grads_rnn(x, h, gr, ws=ws)
e1.record()
torch.cuda.synchronize()
print(f"wgrad {e0.elapsed_time(e1) / 40:.3f} ms")
