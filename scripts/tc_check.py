#!/usr/bin/env python
"""Development check: tensor-core level-0 fold vs the FFMA fold vs the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bppsa_workloads as W  # noqa: E402
from oracle import bp  # noqa: E402
from paper_1907_10134_b200 import api  # noqa: E402


def main():
    for (T, B, seed) in ((5, 2, 0), (200, 3, 1), (4096, 16, 2)):
        f = W.norm_preserving_rnn(T, B, 64, seed=seed)
        h, Wm, g = (torch.from_numpy(f[k]).cuda() for k in ("h", "W_hh", "g"))
        jac = api.jacobians_rnn(h, Wm)
        ref, _ = bp.bp_rnn(f["h"], f["W_hh"], f["g"])
        out = {}
        for impl in ("ffma", "tensor", "tensor_tf32"):
            grad, gi = api.scan(jac, g, grad_h_init=True, leaf_impl=impl)
            torch.cuda.synchronize()
            out[impl] = grad.cpu().numpy()
            err = np.abs(out[impl] - ref).max() / np.abs(ref).max()
            print(f"T={T} B={B} {impl}: rel err {err:.3e}", flush=True)
        print("  tensor vs ffma max diff", np.abs(out["tensor"] - out["ffma"]).max(), flush=True)
    for (T, B, seed) in ((300, 3, 1), (5000, 16, 2)):
        w = W.rnn_workload(T, B, 64, seed=seed)
        h, Wm, g = (torch.from_numpy(a).cuda() for a in (w.h, w.W_hh, w.g))
        jac = api.jacobians_rnn(h, Wm)
        ref, _ = bp.bp_rnn(w.h, w.W_hh, w.g)
        for impl in ("ffma", "tensor", "tensor_tf32"):
            for C0 in (64, 256):
                grad, gi = api.scan(jac, g, grad_h_init=True, leaf_impl=impl, block0=C0)
                torch.cuda.synchronize()
                err = np.abs(grad.cpu().numpy() - ref).max() / np.abs(ref).max()
                print(f"realistic T={T} B={B} C0={C0} {impl}: rel err {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
