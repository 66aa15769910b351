"""One full-size (config 4) RNN weight-gradient call, for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_10134_b200 import api
T, B, H = 1 << 20, 16, 64
g0 = torch.Generator(device="cuda").manual_seed(0)
h = torch.rand((T, B, H), device="cuda", generator=g0) * 1.6 - 0.8
gr = torch.randn((T, B, H), device="cuda", generator=g0)
x = (torch.rand((T, B, 1), device="cuda", generator=g0) < 0.5).float()
ws = api.workspace(api.weight_grads_workspace_size(T, B, H, 1))
for _ in range(2):
    api.weight_grads_rnn(x, h, gr, ws=ws)
torch.cuda.synchronize()
