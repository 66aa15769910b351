"""Dev aid: quick parity check of the level-0 engines (int8 / 3xFP16 / FFMA)
against the fp64 oracle on the realistic and norm-preserving RNN families.

    python scripts/i8_check.py [T ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bppsa_workloads as W  # noqa: E402
from oracle import bp  # noqa: E402
from paper_1907_10134_b200 import api  # noqa: E402


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel(got, ref):
    got = got.cpu().numpy().astype(np.float64)
    return float(np.abs(got - ref).max() / np.abs(ref).max())


def run(h, Wm, g, **kw):
    jac = api.jacobians_rnn(cu(h), cu(Wm))
    grad, gi = api.scan(jac, cu(g), grad_h_init=True, **kw)
    torch.cuda.synchronize()
    return grad, gi


def main():
    Ts = [int(a) for a in sys.argv[1:]] or [100, 1000, 4096]
    for T in Ts:
        for fam in ("real", "norm"):
            if fam == "real":
                w = W.rnn_workload(T, 16, 64, seed=T)
                h, Wm, g = w.h, w.W_hh, w.g
            else:
                f = W.norm_preserving_rnn(T, 16, 64, seed=T)
                h, Wm, g = f["h"], f["W_hh"], f["g"]
            t0 = time.time()
            ref, ref_init = bp.bp_rnn(h, Wm, g)
            to = time.time() - t0
            out = []
            for impl in ("int8", "tensor", "ffma"):
                for blocks in ((0, 0), (512, 32), (64, 8)):
                    if T < 1000 and blocks[0] == 512:
                        continue
                    grad, gi = run(h, Wm, g, leaf_impl=impl, block0=blocks[0], block=blocks[1])
                    out.append(f"{impl}{blocks}={rel(grad, ref):.2e}")
            print(f"T={T} {fam} (oracle {to:.1f}s): " + " ".join(out), flush=True)


if __name__ == "__main__":
    main()
