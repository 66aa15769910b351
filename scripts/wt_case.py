import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import bppsa_workloads as W
from paper_1907_10134_b200 import api
T, B, b0, b1 = map(int, sys.argv[1:5])
impl = sys.argv[5] if len(sys.argv) > 5 else "int8"
f = W.norm_preserving_rnn(T, B, 64, seed=3)
jac = api.jacobians_rnn(torch.from_numpy(f["h"]).cuda(), torch.from_numpy(f["W_hh"]).cuda())
g, gi = api.scan(jac, torch.from_numpy(f["g"]).cuda(), grad_h_init=True, block0=b0, block=b1, leaf_impl=impl)
torch.cuda.synchronize()
print("ok", T, B, b0, b1, flush=True)
