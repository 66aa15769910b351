"""Dev aid: max-norm relative error of the default (int8) and FFMA engines on
the norm-preserving family (H = 64, B = 4) at several T, for A/B of fold
arithmetic variants.  python scripts/prec_ab.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bppsa_workloads as W  # noqa: E402
from oracle import bp  # noqa: E402
from paper_1907_10134_b200 import api  # noqa: E402


def rel(g, ref):
    g = g.cpu().numpy().astype(np.float64)
    return float(np.abs(g - ref).max() / np.abs(ref).max())


for T in [int(a) for a in (sys.argv[1:] or ["4096", "16384", "65536"])]:
    f = W.norm_preserving_rnn(T, 4, 64, seed=7)
    ref, _ = bp.bp_rnn(f["h"], f["W_hh"], f["g"])
    jac = api.jacobians_rnn(torch.from_numpy(f["h"]).cuda(), torch.from_numpy(f["W_hh"]).cuda())
    g = torch.from_numpy(f["g"]).cuda()
    out = []
    for impl in ("int8", "ffma"):
        for bl in ((0, 0), (512, 32), (1024, 32)):
            gr, _ = api.scan(jac, g, grad_h_init=True, block0=bl[0], block=bl[1], leaf_impl=impl)
            torch.cuda.synchronize()
            out.append(f"{impl}{bl}={rel(gr, ref):.2e}")
    print(f"T={T}:", " ".join(out), flush=True)
