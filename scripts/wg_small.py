import os, sys
os.environ["BPPSA_FORCE_TC_WGRAD"] = "1"
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bp
from paper_1907_10134_b200 import api
rng = np.random.default_rng(0)
for T, B in ((2, 16), (4, 16), (1, 32), (64, 16), (66, 16), (130, 16), (1024, 16), (1030, 16), (3000, 16)):
    H = 64
    h = rng.uniform(-0.9, 0.9, (T, B, H)).astype(np.float32)
    g = rng.standard_normal((T, B, H)).astype(np.float32)
    x = rng.standard_normal((T, B, 1)).astype(np.float32)
    r = bp.weight_grads_rnn(x, h, g)
    out = api.weight_grads_rnn(torch.from_numpy(x).cuda(), torch.from_numpy(h).cuda(), torch.from_numpy(g).cuda())
    got = out[1].cpu().numpy()
    print(T * B, "rows: dW_hh rel", np.abs(got - r[1]).max() / np.abs(r[1]).max(), flush=True)

# timing at config-4 size: tensor path (force=1 in this process)
T, B, H = 1 << 20, 16, 64
g0 = torch.Generator(device="cuda").manual_seed(0)
h = torch.rand((T, B, H), device="cuda", generator=g0) * 1.6 - 0.8
gr = torch.randn((T, B, H), device="cuda", generator=g0)
x = (torch.rand((T, B, 1), device="cuda", generator=g0) < 0.5).float()
ws = api.workspace(api.weight_grads_workspace_size(T, B, H, 1))
out = api.weight_grads_rnn(x, h, gr, ws=ws)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    api.weight_grads_rnn(x, h, gr, ws=ws)
e1.record()
torch.cuda.synchronize()
print("tc wgrad ms", e0.elapsed_time(e1) / 5)
# fp64 check of dW_hh on a slice of rows via torch (independent of both paths)
d = ((1 - h.double() ** 2) * gr.double()).reshape(-1, H)
hp = torch.cat([torch.zeros(B, H, device="cuda", dtype=torch.float64), h.double().reshape(-1, H)[:-B]])
ref = d.T @ hp
print("full-size dW_hh rel", ((out[1].double() - ref).abs().max() / ref.abs().max()).item())
