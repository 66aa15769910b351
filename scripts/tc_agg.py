#!/usr/bin/env python
"""Dev aid: compare level-1 block aggregates (workspace) of the tensor and FFMA
level-0 folds against fp64 products."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bppsa_workloads as W  # noqa: E402
from oracle import bp  # noqa: E402
from paper_1907_10134_b200 import api  # noqa: E402


def main():
    H = 64
    for C0 in (2, 4, 8, 16, 64):
        T, B = 3 * C0 - 1, 4          # S = 3*C0: head block + 2 matrix blocks
        f = W.norm_preserving_rnn(T, B, H, seed=C0)
        h, Wm, g = (torch.from_numpy(f[k]).cuda() for k in ("h", "W_hh", "g"))
        jac = api.jacobians_rnn(h, Wm)
        res = {}
        for impl in ("ffma", "tensor"):
            ws = api.workspace(api.scan_workspace_size(jac, "blocked", C0, 2))
            ws.zero_()
            api.scan(jac, g, ws=ws, block0=C0, block=2, leaf_impl=impl)
            torch.cuda.synchronize()
            agg = ws[: B * 3 * H * H * 4].view(torch.float32).view(B, 3, H, H).cpu().numpy()   # [b][q][col j][row i]
            res[impl] = agg
        # fp64 reference of block q (slots q*C0 .. q*C0+C0-1, times T - s): agg = a[s_end] ... a[s_start]
        JT = np.stack([bp.rnn_jt(f["h"][t], f["W_hh"]) for t in range(T)])
        for q in (1, 2):
            P = np.broadcast_to(np.eye(H), (B, H, H)).copy()
            for s in range(q * C0, q * C0 + C0):
                P = np.einsum("bij,bjk->bik", JT[T - s], P)
            for impl in ("ffma", "tensor"):
                got = res[impl][:, q].transpose(0, 2, 1)      # column-major -> [b][i][j]
                err = np.abs(got - P).max() / np.abs(P).max()
                print(f"C0={C0:3d} q={q} {impl:6s}: rel err {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
