"""Pins for oracle/csr.py: values printed in the paper (Table 1) and SPEC,
dense brute force (torch.autograd Jacobians, dense matmul), exhaustive
structural counts."""
import json
import math
import os

import numpy as np
import pytest
import torch

import bppsa_workloads as W
from oracle import csr as C, scan as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
RNG = np.random.default_rng(77)


def _round(x, d):
    return float(f"{x:.{d}f}")


def test_table1_sparsity_and_sizes():
    """Table 1 and the 768 MB / 6.5 MB figures."""
    t = GOLD["table1_sparsity"]
    c1 = t["conv1"]
    m = C.conv_tjac_exact(c1["ci"], c1["co"], c1["h"], c1["w"])
    C.check(m)
    rows, cols = m.rows, m.cols
    assert (rows, cols) == (3 * 32 * 32, 64 * 32 * 32)
    assert _round(1 - m.nnz / (rows * cols), c1["digits"]) == c1["printed"]
    mb = GOLD["conv1_memory_MB"]
    assert rows * cols * mb["bytes_per_value"] / 2 ** 20 == mb["dense_MB"]
    assert round(m.nnz * mb["bytes_per_value"] / 2 ** 20, 1) == mb["csr_MB"]
    r1 = t["relu1"]
    x = RNG.standard_normal(r1["c"] * r1["h"] * r1["w"])
    rm = C.relu_tjac(x)
    assert _round(1 - rm.nnz / (rm.rows * rm.cols), r1["digits"]) == r1["printed"]
    p1 = t["pool1"]
    c, h, w = p1["c"], p1["h"], p1["w"]
    pidx = _pool_indices(RNG.standard_normal((c, h, w)))
    pm = C.maxpool_window_tjac(pidx, c, h, w)
    assert _round(1 - pm.nnz / (pm.rows * pm.cols), p1["digits"]) == p1["printed"]
    # Table 1's closed forms
    assert 1 - rm.nnz / (rm.rows * rm.cols) == pytest.approx(1 - 1 / (c * h * w), abs=1e-15)
    assert 1 - pm.nnz / (pm.rows * pm.cols) == pytest.approx(1 - 4 / (c * h * w), abs=1e-15)
    # Alg. 3's padded allocation 3w(3h-2) c_i c_o
    assert 3 * 32 * (3 * 32 - 2) * 3 * 64 == 1732608


def _pool_indices(x):
    t = torch.from_numpy(x)[None]
    _, idx = torch.nn.functional.max_pool2d(t, 2, 2, return_indices=True)
    return idx[0].numpy()


def _conv_dense_jt(ci, co, h, w, Wt):
    x = torch.zeros(ci * h * w, dtype=torch.float64)
    f = lambda v: torch.nn.functional.conv2d(v.view(1, ci, h, w), torch.from_numpy(Wt), padding=1).reshape(-1)
    return torch.autograd.functional.jacobian(f, x).numpy().T


@pytest.mark.parametrize("ci,co,h,w", [(1, 1, 3, 3), (2, 3, 4, 5), (3, 2, 5, 3), (2, 2, 6, 4)])
def test_conv_algs_2_to_4_vs_autograd(ci, co, h, w):
    Wt = RNG.standard_normal((co, ci, 3, 3))
    ref = _conv_dense_jt(ci, co, h, w, Wt)
    a = C.conv_tjac_algs(ci, co, h, w, Wt)
    C.check(a)
    assert a.nnz == 3 * w * (3 * h - 2) * ci * co          # Alg. 3 allocation
    assert np.array_equal(C.to_dense(a), ref)
    e = C.conv_tjac_exact(ci, co, h, w, Wt)
    assert np.array_equal(C.to_dense(e), ref)


@pytest.mark.parametrize("ci,co,h,w", [(2, 2, 2, 2), (1, 3, 1, 1), (3, 1, 2, 5), (2, 4, 1, 4)])
def test_conv_exact_small_maps_vs_autograd(ci, co, h, w):
    """VGG-11 conv7/conv8 run at 2x2 (and 1x1 would be legal): generic stencil."""
    Wt = RNG.standard_normal((co, ci, 3, 3))
    e = C.conv_tjac_exact(ci, co, h, w, Wt)
    C.check(e)
    assert np.array_equal(C.to_dense(e), _conv_dense_jt(ci, co, h, w, Wt))


def test_conv_nnz_exhaustive():
    for h in range(2, 9):
        for w in range(2, 9):
            for ci in range(1, 4):
                for co in range(1, 4):
                    m = C.conv_tjac_exact(ci, co, h, w)
                    assert m.nnz == ci * co * (3 * h - 2) * (3 * w - 2)
                    if h >= 3 and w >= 3 and ci * co <= 2:
                        a = C.conv_tjac_algs(ci, co, h, w, np.ones((co, ci, 3, 3)))
                        assert a.nnz == 3 * w * (3 * h - 2) * ci * co
                        assert int((a.data != 0).sum()) == m.nnz


def test_conv_pruned_pattern_drops_zero_taps():
    Wt = RNG.standard_normal((3, 2, 3, 3))
    Wt[RNG.random(Wt.shape) < 0.7] = 0.0
    e = C.conv_tjac_exact(2, 3, 5, 4, Wt, drop_zero_weights=True)
    C.check(e)
    assert not (e.data == 0).any()
    assert np.array_equal(C.to_dense(e), _conv_dense_jt(2, 3, 5, 4, Wt))


def test_relu_tjac():
    """Algs. 5-7 vs central differences away from the kink (strict x > 0)."""
    x = RNG.standard_normal(50)
    x[3] = 0.0
    m = C.relu_tjac(x)
    C.check(m)
    D = C.to_dense(m)
    assert np.array_equal(D, np.diag((x > 0).astype(float)))
    assert D[3, 3] == 0.0


def test_maxpool_tjac_vs_autograd():
    c, h, w = 3, 6, 4
    x = RNG.standard_normal((c, h, w))
    pidx = _pool_indices(x)
    xt = torch.from_numpy(x).reshape(-1)
    f = lambda v: torch.nn.functional.max_pool2d(v.view(1, c, h, w), 2, 2).reshape(-1)
    ref = torch.autograd.functional.jacobian(f, xt).numpy().T
    a = C.maxpool_tjac(pidx, c, h, w)
    C.check(a)
    assert np.array_equal(C.to_dense(a), ref)
    win = C.maxpool_window_tjac(pidx, c, h, w)
    C.check(win)
    assert np.array_equal(C.to_dense(win), ref)
    assert win.nnz == c * h * w and a.nnz == c * (h // 2) * (w // 2)


def test_spec_examples():
    e = GOLD["spgemm_example"]
    A, B = C.from_dense(np.array(e["A"], float)), C.from_dense(np.array(e["B"], float))
    assert np.array_equal(C.to_dense(C.spgemm(A, B)), np.array(e["AB"], float))
    I3 = C.from_dense(np.eye(3))
    M = C.from_dense(RNG.integers(-3, 4, (3, 3)).astype(float))
    P = C.spgemm(I3, M)
    assert np.array_equal(P.indptr, M.indptr) and np.array_equal(P.indices, M.indices)
    assert np.array_equal(P.data, M.data)
    e = GOLD["spmv_example"]
    assert C.spmv(C.from_dense(np.array(e["A"], float)), np.array(e["v"], float)).tolist() == e["Av"]
    Z = C.CSR(8, 8, np.zeros(9, np.int64), np.zeros(0, np.int64), np.zeros(0))
    assert not C.spmv(Z, RNG.standard_normal(8)).any()


@pytest.mark.parametrize("seed", range(10))
def test_plan_vs_dense(seed):
    """plan_product pattern == boolean dense product; execute_plan == dense
    matmul; one plan reused for many data variants."""
    rng = np.random.default_rng(seed)
    m, k, n = rng.integers(1, 33, 3)
    ka, kb = rng.random((m, k)) < 0.15, rng.random((k, n)) < 0.15
    A = C.from_dense(np.where(ka, rng.standard_normal((m, k)), 0), keep=ka)
    B = C.from_dense(np.where(kb, rng.standard_normal((k, n)), 0), keep=kb)
    plan = C.plan_product(A.pattern(), B.pattern())
    C.check(plan.out)
    assert np.array_equal(C.to_dense(C.CSR(m, n, plan.out.indptr, plan.out.indices,
                                             np.ones(plan.out.nnz))) != 0,
                          (ka.astype(int) @ kb.astype(int)) > 0)
    for _ in range(5):
        ad, bd = rng.standard_normal(A.nnz), rng.standard_normal(B.nnz)
        out = C.execute_plan(plan, ad, bd)
        Ad = C.to_dense(C.CSR(m, k, A.indptr, A.indices, ad))
        Bd = C.to_dense(C.CSR(k, n, B.indptr, B.indices, bd))
        got = C.to_dense(C.CSR(m, n, plan.out.indptr, plan.out.indices, out))
        assert np.allclose(got, Ad @ Bd, rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        C.plan_product(A.pattern(), C.from_dense(np.ones((int(k) + 1, 2))))


def _small_vgg(B=2, seed=0):
    cfg = [4, "M", 6, 6, "M", 8, "M"]
    rng = np.random.default_rng(seed)
    ws, c = [], 3
    for v in cfg:
        if v != "M":
            w = rng.standard_normal((v, c, 3, 3)) * 0.4
            w[rng.random(w.shape) < 0.5] = 0.0
            ws.append(w.astype(np.float32))
            c = v
    imgs = rng.standard_normal((B, 3, 8, 8)).astype(np.float32)
    return cfg, ws, imgs


def csr_chain(cfg, ws, recs, hw, B):
    """Transposed-Jacobian chain J_1^T..J_n^T (time order) of a conv stack."""
    ops = W.vgg11_ops(cfg, 3, hw)
    chain, wi = [], 0
    for op, rec in zip(ops, recs):
        kind = op[0]
        if kind == "conv":
            _, ci, co, h, w = op
            chain.append(C.conv_tjac_exact(ci, co, h, w, ws[wi], drop_zero_weights=True))
            wi += 1
        elif kind == "relu":
            _, c, h, w = op
            ms = [C.relu_tjac(rec[1][b]) for b in range(B)]
            chain.append(C.CSR(ms[0].rows, ms[0].cols, ms[0].indptr, ms[0].indices,
                               np.stack([m.data for m in ms])))
        else:
            _, c, h, w = op
            ms = [C.maxpool_window_tjac(rec[1][b], c, h, w) for b in range(B)]
            chain.append(C.CSR(ms[0].rows, ms[0].cols, ms[0].indptr, ms[0].indices,
                               np.stack([m.data for m in ms])))
    return chain


def test_csr_chain_bp_and_hybrid_vs_autograd():
    """Config-5 semantics on a reduced VGG: sequential SpMV chain (eqn:backprop)
    and the hybrid CSR scan reproduce torch.autograd's VJPs through the
    whole conv stack (fp64)."""
    B = 2
    cfg, ws, imgs = _small_vgg(B)
    recs, out = W.vgg11_forward(imgs, ws, cfg)
    chain = csr_chain(cfg, ws, recs, 8, B)
    seed = np.random.default_rng(9).standard_normal((B, out[0].size))
    # torch reference: gradient of <seed, f(x)> w.r.t. every intermediate x_i
    x = torch.from_numpy(imgs.astype(np.float64)).requires_grad_(True)
    acts, cur, wi = [x], x, 0
    for v in cfg:
        if v == "M":
            cur = torch.nn.functional.max_pool2d(cur, 2, 2)
            cur.retain_grad(); acts.append(cur)
        else:
            cur = torch.nn.functional.conv2d(cur, torch.from_numpy(ws[wi].astype(np.float64)), padding=1)
            cur.retain_grad(); acts.append(cur)
            cur = torch.relu(cur)
            cur.retain_grad(); acts.append(cur)
            wi += 1
    (cur.reshape(B, -1) * torch.from_numpy(seed)).sum().backward()
    n = len(chain)
    # sequential BP: grad x_{i-1} = J_i^T grad x_i
    v = seed
    grads = {n: v}
    for i in range(n, 0, -1):
        v = C.spmv(chain[i - 1], v)
        grads[i - 1] = v
    for i in range(n + 1):
        ref = acts[i].grad.reshape(B, -1).numpy()
        assert np.allclose(grads[i], ref, rtol=1e-12, atol=1e-12), i
    # hybrid / Alg. 1 over CSR elements (scan order: seed, J_n^T, ..., J_1^T)
    a = [S.El("v", seed)] + [S.El("s", chain[n - k]) for k in range(1, n + 1)]
    L = S.num_levels(n)
    for u, dl in ((0, 0), (2, 3), (L - 1, L), (min(3, L - 1), min(4, L))):
        res = S.hybrid(a, u, dl)
        for k in range(1, n + 1):
            assert np.allclose(res[k].val, grads[n - k + 1], rtol=1e-12, atol=1e-12), (u, dl, k)


def test_mfcc_shapes_golden():
    """Table 3: F = 1 + floor(132300 / hop), C = 2 (n_mfcc - 1) (reading P8);
    the generator's IRMAS_SETS carry exactly these shapes."""
    g = GOLD["mfcc_shapes"]
    for name in ("S", "M", "L"):
        e = g[name]
        assert 1 + g["clip_samples"] // e["hop"] == e["F"]
        assert 2 * (e["n_mfcc"] - 1) == e["C"]
        assert W.IRMAS_SETS[name] == (e["F"], e["C"])
