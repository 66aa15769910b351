"""C5 hybrid (2, 3) CSR scan once (dev aid for ncu captures of spgemm_kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bppsa_workloads as W  # noqa: E402
from paper_1907_10134_b200 import api  # noqa: E402
from paper_1907_10134_b200.vgg import CsrChain  # noqa: E402

w = W.vgg11_workload(B=16, seed=0)
relu_in = [torch.from_numpy(r[1]).cuda() for r in w["recs"] if r[0] == "relu"]
pools = [torch.from_numpy(r[1]).cuda() for r in w["recs"] if r[0] == "pool"]
chain = CsrChain(W.VGG11_CFG, w["weights"], relu_in, pools)
seed = torch.from_numpy(w["g"]).cuda()
plan = chain.plan(2, 3)
ws = api.workspace(plan.workspace_size(16, chain.batched))
grads = [torch.empty((16, d), device="cuda") for d in plan.dims]
for _ in range(2):
    api.csr_scan(plan, chain.data, chain.batched, seed, grads=grads, ws=ws)
torch.cuda.synchronize()
print("ok")
