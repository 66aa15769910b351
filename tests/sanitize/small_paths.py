"""Small runs of every hand-written kernel family, for compute-sanitizer
(tests/test_gpu_sanitizer.py): the exact-integer fold and walk, the 3xFP16 /
3xTF32 folds and the TMA walk, the CUDA-core leaves and levels, the tcgen05
weight gradients, the GRU path, the affine scan, the CSR SpGEMM scan and the
peer-exchange kernels and the publish fused into the shard up-sweep (one rank).  Exits non-zero on a wrong result."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bppsa_workloads as W  # noqa: E402
from paper_1907_10134_b200 import api  # noqa: E402


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    T, B, H = 300, 5, 64
    w = W.rnn_workload(T, B, H, seed=3)
    jac = api.jacobians_rnn(cu(w.h), cu(w.W_hh))
    outs = {}
    for impl in ("int8", "tensor", "tensor_tf32", "ffma"):
        g, gi = api.scan(jac, cu(w.g), grad_h_init=True, block0=64, block=8, leaf_impl=impl)
        outs[impl] = g
    api.scan(jac, cu(w.g), mode="linear")
    api.weight_grads_rnn(cu(w.x), cu(w.h), outs["int8"])
    e = torch.randn((T, B, H), device="cuda") * 0.01
    api.scan_affine(jac, cu(w.g), e, block0=64, block=8)
    # GRU (H = 20)
    gw = W.gru_workload("S", 4, seed=1)
    tape = {k: cu(v) for k, v in gw.tape.items()}
    jg = api.jacobians_gru(tape["h_prev"], tape["r"], tape["z"], tape["n"], tape["M"], cu(gw.params["W_hh3"]))
    gg, _ = api.scan(jg, cu(gw.g), block0=16, block=16)
    api.weight_grads_gru(cu(gw.x), tape, gg)
    # CSR SpGEMM scan: a small random chain, full Alg. 1 schedule
    rng = np.random.default_rng(0)
    n, Bc = 6, 3
    dims = rng.integers(5, 30, n + 1)
    pats, data, batched = [], [], []
    for k in range(n):
        keep = rng.random((dims[k], dims[k + 1])) < 0.3
        indptr = np.concatenate([[0], np.cumsum(keep.sum(axis=1))]).astype(np.int64)
        indices = np.nonzero(keep)[1].astype(np.int32)
        pats.append((int(dims[k]), int(dims[k + 1]), indptr, indices))
        data.append(torch.randn(int(keep.sum()), device="cuda"))
        batched.append(0)
    plan = api.csr_plan_create(pats, 2, 3)
    api.csr_scan(plan, data, batched, torch.randn((Bc, int(dims[n])), device="cuda"))
    # peer exchange, one rank on one device
    n = B * H * H
    mail = torch.zeros((2, 1, n), device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    acks = torch.zeros(1, dtype=torch.int32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    mp = torch.tensor([mail.data_ptr()], dtype=torch.int64, device="cuda")
    fp = torch.tensor([flags.data_ptr()], dtype=torch.int64, device="cuda")
    ap = torch.tensor([acks.data_ptr()], dtype=torch.int64, device="cuda")
    agg = torch.randn(n, device="cuda")
    for ep in (1, 2, 3):
        api.exchange_publish(agg, 0, 1, mp, fp, counter, acks, ep)
        api.exchange_wait(flags, 0, 1, ep)
        api.exchange_ack(0, 1, ap, ep)
    torch.cuda.synchronize()
    if not torch.equal(mail[1, 0], agg):
        sys.exit(3)
    # the publish fused into the shard up-sweep's top level (epochs 4, 5)
    ws = api.workspace(api.scan_workspace_size(jac, "blocked", 64, 8))
    ref_agg = torch.empty(n, device="cuda")
    api.scan_shard_up(jac, cu(w.g), ref_agg, ws, 64, 8)
    agg2 = torch.empty(n, device="cuda")
    for ep in (4, 5):
        api.scan_shard_up_publish(jac, cu(w.g), agg2, ws, 0, 1, mp, fp, counter, acks, ep, 64, 8)
        api.exchange_wait(flags, 0, 1, ep)
        api.exchange_ack(0, 1, ap, ep)
    torch.cuda.synchronize()
    if not torch.equal(mail[1, 0, :H * 1], ref_agg[:H]) or not torch.equal(agg2[:H], ref_agg[:H]):
        sys.exit(4)
    ref = outs["ffma"].cpu().numpy()
    for impl in ("int8", "tensor", "tensor_tf32"):
        err = float(np.abs(outs[impl].cpu().numpy() - ref).max() / np.abs(ref).max())
        if not err < 1e-4:
            print(f"{impl}: rel err {err:.2e}")
            sys.exit(2)
    print("small paths ok")


if __name__ == "__main__":
    main()
