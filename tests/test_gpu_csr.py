"""GPU parity of the CSR SpGEMM hybrid scan (config 5)
against the oracle's sequential SpMV chain (eqn:backprop) and CSR builders."""
import numpy as np
import pytest
import torch

import bppsa_workloads as W
from oracle import csr as C, scan as S

pytestmark = pytest.mark.gpu


def rel(got, ref):
    got = got.detach().cpu().numpy().astype(np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def seq_bp(chain, seed):
    """Oracle: sequential BP grad x_{k-1} = J_k^T grad x_k (returns k = 0..n)."""
    n = len(chain)
    out = [None] * (n + 1)
    v = np.asarray(seed, np.float64)
    out[n] = v
    for k in range(n, 0, -1):
        v = C.spmv(chain[k - 1], v)
        out[k - 1] = v
    return out


def random_chain(n, B, seed, int_data):
    rng = np.random.default_rng(seed)
    dims = rng.integers(5, 40, n + 1)
    chain, pats, data, batched = [], [], [], []
    for k in range(n):
        keep = rng.random((dims[k], dims[k + 1])) < 0.25
        bat = int(rng.random() < 0.5)
        shape = (B, keep.sum()) if bat else (keep.sum(),)
        vals = (rng.integers(-1, 2, shape) if int_data else rng.standard_normal(shape) * 0.5).astype(np.float32)
        m = C.from_dense(np.zeros(keep.shape), keep=keep)
        m.data = vals.astype(np.float64)
        chain.append(m)
        pats.append((int(dims[k]), int(dims[k + 1]), m.indptr, m.indices.astype(np.int32)))
        data.append(torch.from_numpy(np.ascontiguousarray(vals.T if bat else vals)).cuda())   # [nnz, B]
        batched.append(bat)
    s = (rng.integers(-2, 3, (B, dims[n])) if int_data else rng.standard_normal((B, dims[n]))).astype(np.float32)
    return chain, pats, data, batched, s


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 9, 13])
def test_random_chains_all_schedules_bit_exact(lib, n):
    B = 3
    chain, pats, data, batched, s = random_chain(n, B, seed=n, int_data=True)
    ref = seq_bp(chain, s)
    assert max(np.abs(r).max() for r in ref) < 2 ** 24
    L = S.num_levels(n)
    for u in range(0, L):
        for dl in (u, u + 1):
            if dl > L:
                continue
            plan = lib.csr_plan_create(pats, u, dl)
            grads = lib.csr_scan(plan, data, batched, torch.from_numpy(s).cuda())
            torch.cuda.synchronize()
            for k in range(n + 1):
                assert np.array_equal(grads[k].cpu().numpy(), ref[k]), (u, dl, k)


@pytest.mark.parametrize("n", [4, 11])
def test_random_chains_float(lib, n):
    B = 4
    chain, pats, data, batched, s = random_chain(n, B, seed=100 + n, int_data=False)
    ref = seq_bp(chain, s)
    scale = max(np.abs(r).max() for r in ref[1:])
    plan = lib.csr_plan_create(pats, S.num_levels(n) - 1, S.num_levels(n))      # full Alg. 1
    grads = lib.csr_scan(plan, data, batched, torch.from_numpy(s).cuda())
    for k in range(1, n + 1):
        assert np.abs(grads[k].cpu().numpy() - ref[k]).max() <= 1e-5 * scale


def test_schedule_errors(lib):
    chain, pats, data, batched, s = random_chain(5, 2, seed=1, int_data=True)
    with pytest.raises(lib.BppsaError, match="INVALID_ARGUMENT"):
        lib.csr_plan_create(pats, 1, 3)
    with pytest.raises(lib.BppsaError, match="SHAPE"):
        bad = list(pats)
        bad[2] = (bad[2][0] + 1,) + bad[2][1:]
        lib.csr_plan_create(bad, 0, 0)
    with pytest.raises(lib.BppsaError, match="NOT_SUPPORTED"):
        lib.csr_plan_create(pats, 2, 3, max_contributions=1)


def vgg_case(cfg, B, hw, seed, density):
    rng = np.random.default_rng(seed)
    ws, c = [], 3
    for v in cfg:
        if v != "M":
            w = (rng.standard_normal((v, c, 3, 3)) * np.sqrt(2.0 / (9 * v))).astype(np.float32)
            if density < 1:
                k = max(1, int(round(density * w.size)))
                thr = np.partition(np.abs(w).ravel(), w.size - k)[w.size - k]
                w = np.where(np.abs(w) >= thr, w, 0.0).astype(np.float32)
            ws.append(w)
            c = v
    imgs = rng.standard_normal((B, 3, hw, hw)).astype(np.float32)
    recs, out = W.vgg11_forward(imgs, ws, cfg)
    seed_vec = rng.standard_normal((B, out[0].size)).astype(np.float32)
    return ws, recs, seed_vec


def build_both(lib, cfg, ws, recs, B, hw):
    from paper_1907_10134_b200.vgg import CsrChain
    relu_in = [torch.from_numpy(r[1]).cuda() for r in recs if r[0] == "relu"]
    pools = [torch.from_numpy(r[1]).cuda() for r in recs if r[0] == "pool"]
    chain_dev = CsrChain(cfg, ws, relu_in, pools, hw=hw)
    # oracle chain (independent builders)
    ops = W.vgg11_ops(cfg, 3, hw)
    chain, wi = [], 0
    for op, rec in zip(ops, recs):
        if op[0] == "conv":
            _, ci, co, h, w = op
            chain.append(C.conv_tjac_exact(ci, co, h, w, ws[wi], drop_zero_weights=True))
            wi += 1
        elif op[0] == "relu":
            ms = [C.relu_tjac(rec[1][b]) for b in range(B)]
            chain.append(C.CSR(ms[0].rows, ms[0].cols, ms[0].indptr, ms[0].indices, np.stack([m.data for m in ms])))
        else:
            _, c, h, w = op
            ms = [C.maxpool_window_tjac(rec[1][b], c, h, w) for b in range(B)]
            chain.append(C.CSR(ms[0].rows, ms[0].cols, ms[0].indptr, ms[0].indices, np.stack([m.data for m in ms])))
    return chain_dev, chain


def test_builders_data_exact(lib):
    """Device data of the analytical builders == the oracle's (bit-exact)."""
    cfg, B, hw = [4, "M", 6, "M"], 3, 8
    ws, recs, s = vgg_case(cfg, B, hw, seed=3, density=0.5)
    dev, ref = build_both(lib, cfg, ws, recs, B, hw)
    for k, (m, d, bat) in enumerate(zip(ref, dev.data, dev.batched)):
        got = d.cpu().numpy().astype(np.float64)
        want = m.data.T if bat else m.data
        assert np.array_equal(got, want), k
        assert np.array_equal(dev.patterns[k][2], m.indptr) and np.array_equal(dev.patterns[k][3], m.indices)


@pytest.mark.parametrize("sched", [(0, 0), (1, 1), (1, 2), (2, 2), (2, 3), (3, 3), (3, 4)])
def test_small_vgg_schedules(lib, sched):
    cfg, B, hw = [4, "M", 6, 6, "M", 8, "M"], 2, 8
    ws, recs, s = vgg_case(cfg, B, hw, seed=7, density=0.5)
    dev, chain = build_both(lib, cfg, ws, recs, B, hw)
    ref = seq_bp(chain, s)
    plan = dev.plan(*sched)
    grads = lib.csr_scan(plan, dev.data, dev.batched, torch.from_numpy(s).cuda())
    torch.cuda.synchronize()
    for k in range(len(chain) + 1):
        assert rel(grads[k], ref[k]) <= 1e-5, (sched, k)


@pytest.mark.slow
@pytest.mark.parametrize("sched", [(1, 2), (2, 3)])
def test_vgg11_config5(lib, sched):
    """Config 5 at full size: VGG-11 conv stack, 32x32x3, B = 16, 97 % pruned."""
    w = W.vgg11_workload(B=16, seed=0)
    cfg, B = W.VGG11_CFG, 16
    dev, chain = build_both(lib, cfg, w["weights"], w["recs"], B, 32)
    ref = seq_bp(chain, w["g"])
    plan = dev.plan(*sched)
    info = plan.info()
    print(sched, info)
    grads = lib.csr_scan(plan, dev.data, dev.batched, torch.from_numpy(w["g"]).cuda())
    torch.cuda.synchronize()
    scale = max(np.abs(r).max() for r in ref)
    for k in range(len(chain) + 1):
        assert np.abs(grads[k].cpu().numpy() - ref[k]).max() <= 1e-4 * scale, k
    if sched == (1, 2):     # the only SpGEMM level: contributions = sum of the oracle's plans
        n = len(chain)
        a = [None] + [chain[n - k] for k in range(1, n + 1)]
        tot = 0
        for i in range(2, n, 2):
            tot += len(C.plan_product(a[i + 1].pattern(), a[i].pattern()).left_pos)
        assert info["contributions"] == tot


# ------------------------------------------------------------------ NEXT-3: device builders, static FLOPs
@pytest.mark.parametrize("ci,co,h,w,density", [(3, 64, 32, 32, 1.0), (64, 128, 16, 16, 0.03), (5, 7, 1, 6, 1.0),
                                                (4, 3, 2, 2, 0.5), (2, 5, 7, 3, 0.3), (512, 512, 2, 2, 0.03)])
def test_device_conv_builder_matches_host_and_oracle(lib, ci, co, h, w, density):
    """bppsa_csr_conv3x3_build (Algs. 2-4 on the GPU) == the host builder and
    the oracle's exact stencil, bit for bit (indptr, indices, tap, data)."""
    rng = np.random.default_rng(ci + co + h)
    wt = rng.standard_normal((co, ci, 3, 3)).astype(np.float32)
    drop = density < 1
    if drop:
        wt[rng.random(wt.shape) >= density] = 0.0
    wdev = torch.from_numpy(wt.reshape(-1)).cuda()
    ip, ix, tap, data = lib.csr_conv3x3_build(ci, co, h, w, wdev, drop_zero=drop, with_data=True)
    torch.cuda.synchronize()
    hip, hix, htap = lib.csr_conv3x3_pattern(ci, co, h, w, wt, drop_zero=drop)
    assert np.array_equal(ip.cpu().numpy(), hip)
    assert np.array_equal(ix.cpu().numpy(), hix)
    assert np.array_equal(tap.cpu().numpy(), htap)
    assert np.array_equal(data.cpu().numpy(), wt.reshape(-1)[htap])
    if ci * co * h * w <= 64 * 128 * 16 * 16:
        m = C.conv_tjac_exact(ci, co, h, w, wt, drop_zero_weights=drop)
        assert np.array_equal(ip.cpu().numpy(), m.indptr) and np.array_equal(ix.cpu().numpy(), m.indices)
        assert np.array_equal(data.cpu().numpy().astype(np.float64), m.data)


def test_device_pool_and_identity_builders(lib):
    for c, h, w in [(64, 32, 32), (3, 2, 2), (5, 6, 4)]:
        ip, ix = lib.csr_maxpool_build(c, h, w)
        hip, hix = lib.csr_maxpool_pattern(c, h, w)
        assert np.array_equal(ip.cpu().numpy(), hip) and np.array_equal(ix.cpu().numpy(), hix)
    ip, ix = lib.csr_identity_build(65536)
    assert np.array_equal(ip.cpu().numpy(), np.arange(65537)) and np.array_equal(ix.cpu().numpy(), np.arange(65536))


def _steps_equal(got, want):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g == {k: w[k] for k in g}, (g, w)


@pytest.mark.parametrize("n", [1, 3, 8, 13])
def test_plan_steps_match_oracle_random(lib, n):
    """bppsa_csr_plan_steps == oracle.scan.hybrid_steps on every split."""
    chain, pats, *_ = random_chain(n, 2, seed=40 + n, int_data=True)
    for lv in [(u, dl) for u in range(0, S.num_levels(n)) for dl in (u, u + 1) if dl <= S.num_levels(n)]:
        got = lib.csr_plan_steps(lib.csr_plan_create(pats, *lv))
        _steps_equal(got, S.hybrid_steps([m.pattern() for m in chain], *lv))


def test_plan_steps_small_vgg(lib):
    cfg, B, hw = [4, "M", 6, 6, "M", 8, "M"], 2, 8
    ws, recs, s = vgg_case(cfg, B, hw, seed=7, density=0.5)
    dev, chain = build_both(lib, cfg, ws, recs, B, hw)
    for lv in [(0, 0), (2, 3), (3, 4)]:
        _steps_equal(lib.csr_plan_steps(dev.plan(*lv)), S.hybrid_steps([m.pattern() for m in chain], *lv))
