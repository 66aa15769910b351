"""bppsa_csr_plan_create_symbolic (host only, no GPU): the static FLOP analysis
of a hybrid schedule (fig:prune_symbolic) without contribution
lists, against the oracle's hybrid_steps (explicit structural products,
oracle/csr.plan_product) and the closed-form pair count, and the paper's own
(u, dl) = (3, 4) schedule on the 97 %-pruned VGG-11 (DESIGN reading
22), whose 9.1e10 contribution pairs no numeric plan holds."""
import numpy as np
import pytest

import bppsa_workloads as W
from oracle import csr as C, scan as S


@pytest.fixture(scope="module")
def api():
    from paper_1907_10134_b200 import api as a   # loads libbppsa.so; these calls make no CUDA call
    return a


def random_patterns(n, seed, density=0.25):
    rng = np.random.default_rng(seed)
    dims = rng.integers(5, 40, n + 1)
    chain, pats = [], []
    for k in range(n):
        keep = rng.random((dims[k], dims[k + 1])) < density
        m = C.from_dense(np.zeros(keep.shape), keep=keep)
        chain.append(m)
        pats.append((int(dims[k]), int(dims[k + 1]), m.indptr, m.indices.astype(np.int32)))
    return chain, pats


def splits(n):
    L = S.num_levels(n)
    return [(u, dl) for u in range(0, L) for dl in (u, u + 1) if dl <= L]


def steps_equal(got, want):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g == {k: w[k] for k in g}, (g, w)


@pytest.mark.parametrize("n,density", [(1, 0.25), (3, 0.25), (8, 0.25), (13, 0.25), (21, 0.1), (21, 0.6)])
def test_symbolic_steps_match_oracle_random(api, n, density):
    chain, pats = random_patterns(n, seed=70 + n, density=density)
    for lv in splits(n):
        plan = api.csr_plan_create_symbolic(pats, *lv)
        want = S.hybrid_steps([m.pattern() for m in chain], *lv)
        steps_equal(api.csr_plan_steps(plan), want)
        # info: contributions = sum of the SpGEMM pairs = sum of mm flops / 2
        assert plan.info()["contributions"] == sum(w["flops"] for w in want if w["kind"] == "mm") // 2


def test_symbolic_pairs_closed_form(api):
    """pairs(L R) = sum_k nnz(L[:, k]) nnz(R[k, :]) — counted here from the
    dense 0/1 patterns (a different computation from the library's CSR column
    counts and from the oracle's contribution lists)."""
    chain, pats = random_patterns(3, seed=5, density=0.4)

    def dense(p):
        d = np.zeros((p[0], p[1]), bool)
        for i in range(p[0]):
            d[i, p[3][p[2][i]:p[2][i + 1]]] = True
        return d
    # n = 3: the only level-0 SpGEMM is a[3] <- a[3] a[2] = J_1^T J_2^T
    L, R = dense(pats[0]), dense(pats[1])
    want = int((L.sum(axis=0).astype(np.int64) * R.sum(axis=1)).sum())
    plan = api.csr_plan_create_symbolic(pats, 1, 1)
    mm = [s for s in api.csr_plan_steps(plan) if s["kind"] == "mm"]
    assert len(mm) == 1 and mm[0]["flops"] == 2 * want


def test_symbolic_plan_has_no_numeric_scan(api):
    _, pats = random_patterns(4, seed=3)
    plan = api.csr_plan_create_symbolic(pats, 1, 2)
    with pytest.raises(RuntimeError, match="symbolic"):
        plan.workspace_size(2, [0] * 4)


def vgg_patterns(api, cfg, ws, hw):
    from paper_1907_10134_b200.vgg import conv_stack_ops
    pats, wi = [], 0
    for op in conv_stack_ops(cfg, 3, hw):
        if op[0] == "conv":
            _, ci, co, h, w = op
            ip, ix, _ = api.csr_conv3x3_pattern(ci, co, h, w, np.ascontiguousarray(ws[wi], np.float32), drop_zero=True)
            pats.append((ci * h * w, co * h * w, ip, ix))
            wi += 1
        elif op[0] == "relu":
            _, c, h, w = op
            d = c * h * w
            pats.append((d, d, np.arange(d + 1, dtype=np.int64), np.arange(d, dtype=np.int32)))
        else:
            _, c, h, w = op
            ip, ix = api.csr_maxpool_pattern(c, h, w)
            pats.append((c * h * w, c * (h // 2) * (w // 2), ip, ix))
    return pats


def test_symbolic_small_vgg_matches_oracle(api):
    """A small pruned VGG (the oracle's own conv / ReLU / pool patterns): every
    schedule, the paper's (3, 4) included."""
    cfg, hw = [4, "M", 6, 6, "M", 8, "M"], 8
    rng = np.random.default_rng(11)
    ws, c = [], 3
    for v in cfg:
        if v != "M":
            w = rng.standard_normal((v, c, 3, 3)).astype(np.float32)
            w = np.where(np.abs(w) >= np.quantile(np.abs(w), 0.5), w, 0.0).astype(np.float32)
            ws.append(w)
            c = v
    pats = vgg_patterns(api, cfg, ws, hw)
    ops = W.vgg11_ops(cfg, 3, hw)
    chain, wi = [], 0
    for op in ops:
        if op[0] == "conv":
            _, ci, co, h, w = op
            chain.append(C.conv_tjac_exact(ci, co, h, w, ws[wi], drop_zero_weights=True).pattern())
            wi += 1
        else:
            p = pats[len(chain)]
            chain.append(C.CSR(p[0], p[1], np.asarray(p[2]), np.asarray(p[3]), np.zeros(len(p[3]))).pattern())
    n = len(chain)
    for lv in splits(n):
        steps_equal(api.csr_plan_steps(api.csr_plan_create_symbolic(pats, *lv)), S.hybrid_steps(chain, *lv))


def test_paper_schedule_3_4_on_pruned_vgg11(api):
    """'up-sweep from L0 to L2 ... down-sweep from L7 to L10' = (3, 4)
    on the 97 %-pruned VGG-11 (config 5).  The analysis completes on the host;
    its SpGEMM pair counts equal the closed form from the patterns' column and
    row counts, and the densest product (slots 11..15) has ~9.1e10 pairs."""
    import time
    ws = W.vgg11_pruned_weights(1, 0.03)
    pats = vgg_patterns(api, W.VGG11_CFG, ws, 32)
    t0 = time.perf_counter()
    plan = api.csr_plan_create_symbolic(pats, 3, 4)
    dt = time.perf_counter() - t0
    steps = api.csr_plan_steps(plan)
    mm = [s for s in steps if s["kind"] == "mm"]
    assert [s["level"] for s in mm].count(2) == 2 and len(mm) == 10 + 4 + 2   # slot 0 (the seed) makes the first op of each level an SpMV
    assert max(s["flops"] for s in mm) // 2 == pytest.approx(9.12e10, rel=0.01)
    # level-0 pair counts from the original patterns (column counts x row counts)
    n = len(pats)
    a = [None] + [pats[n - s] for s in range(1, n + 1)]
    lv0 = [s for s in mm if s["level"] == 0]
    k = 0
    for i in range(0, n, 2):
        l, r = i, min(i + 1, n)
        if l == 0:
            continue
        L, R = a[r], a[l]
        colL = np.bincount(np.asarray(L[3]), minlength=L[1])
        rowR = np.diff(np.asarray(R[2]))
        assert lv0[k]["flops"] == 2 * int((colL.astype(np.int64) * rowR).sum())
        k += 1
    print(f"(3, 4) symbolic analysis: {dt:.1f} s, {len(steps)} steps, max SpGEMM pairs {max(s['flops'] for s in mm) // 2:.3g}")
