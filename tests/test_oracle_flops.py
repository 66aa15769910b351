"""Pins for oracle.scan.hybrid_steps, the static FLOP analysis of the CSR
schedule (fig:prune_symbolic; DESIGN reading 23): closed-form
pair counts, dense chains (sparse count = dense complexity), the linear scan
(= the BP baseline), Alg. 1's operation counts (P5: n - L GEMMs, n - 1 GEMVs),
and Table 1's conv1 nnz."""
import numpy as np
import pytest

from oracle import csr as C, scan as S

RNG = np.random.default_rng(5)


def rand_pat(m, n, p):
    return C.from_dense((RNG.random((m, n)) < p).astype(np.float64))


def chain(dims, p):
    return [rand_pat(dims[k], dims[k + 1], p) for k in range(len(dims) - 1)]


def splits(n):
    L = int(n).bit_length()
    return [(u, dl) for u in range(0, max(L - 1, 0) + 1) for dl in (u, u + 1) if dl <= L]


@pytest.mark.parametrize("seed", range(5))
def test_pair_count_closed_form(seed):
    """#contribution pairs of A @ B = sum_k nnz(A[:, k]) nnz(B[k, :])."""
    rng = np.random.default_rng(seed)
    m, k, n = rng.integers(1, 30, 3)
    A = (rng.random((m, k)) < 0.3)
    B = (rng.random((k, n)) < 0.3)
    pl = C.plan_product(C.from_dense(A.astype(float)), C.from_dense(B.astype(float)))
    assert len(pl.left_pos) == int((A.sum(0) * B.sum(1)).sum())
    # and the output pattern is the boolean product
    assert pl.out.nnz == int(((A.astype(int) @ B.astype(int)) > 0).sum())


def test_dense_chain_flops_equal_dense_complexity():
    dims = [4, 6, 5, 7, 3, 6, 5, 4, 6, 3]
    pats = chain(dims, 1.1)                                  # every entry present
    for lv in splits(len(pats)):
        for st in S.hybrid_steps(pats, *lv):
            assert st["flops"] == st["dense_flops"], (lv, st)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 13])
def test_linear_schedule_is_the_bp_baseline(n):
    dims = list(RNG.integers(2, 12, n + 1))
    pats = chain(dims, 0.4)
    st = S.hybrid_steps(pats, 0, 0)
    scan_ops = [s for s in st if s["phase"] != "bp"]
    bp = [s for s in st if s["phase"] == "bp"]
    assert all(s["kind"] == "mv" and s["critical"] for s in scan_ops)
    assert len(scan_ops) == len(bp) == n
    assert sorted(s["flops"] for s in scan_ops) == sorted(s["flops"] for s in bp)
    assert [s["level"] for s in bp] == list(range(n, 0, -1))
    assert sum(s["flops"] for s in bp) == 2 * sum(p.nnz for p in pats)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 8, 21, 33])
def test_alg1_operation_counts(n):
    """Full Alg. 1 = hybrid (L-1, L): n - L SpGEMMs, n - 1 SpMVs (P5), no
    bridge op; exactly one critical op per level."""
    L = int(n).bit_length()
    pats = chain([5] * (n + 1), 0.5)
    st = [s for s in S.hybrid_steps(pats, L - 1, L) if s["phase"] not in ("bp", "extra")]
    assert sum(s["kind"] == "mm" for s in st) == n - L
    assert sum(s["kind"] == "mv" for s in st) == n - 1
    assert not any(s["phase"] == "bridge" for s in st)
    for ph in ("up", "down"):
        for lv in {s["level"] for s in st if s["phase"] == ph}:
            assert sum(s["critical"] for s in st if s["phase"] == ph and s["level"] == lv) == 1


def test_every_split_covers_every_output():
    """Each valid split produces a vector in every slot (asserted inside) and
    one extra op; mm flops never exceed their dense complexity."""
    pats = chain([6, 5, 7, 4, 6, 5, 8, 3, 5, 6, 4, 7], 0.35)
    for lv in splits(len(pats)):
        st = S.hybrid_steps(pats, *lv)
        assert sum(s["phase"] == "extra" for s in st) == 1
        assert all(s["flops"] <= s["dense_flops"] for s in st)


def test_conv1_bp_flops_from_table1_nnz():
    """conv1 (3 -> 64 on 32 x 32): nnz 1,696,512 (Table 1 / P:182), so the BP
    gradient operator costs 2 x 1,696,512 flops per sample."""
    m = C.conv_tjac_exact(3, 64, 32, 32)
    st = S.hybrid_steps([m], 0, 0)
    bp = [s for s in st if s["phase"] == "bp"]
    assert bp[0]["flops"] == 2 * 1_696_512
    assert bp[0]["dense_flops"] == 2 * 3072 * 65536


def test_invalid_split():
    pats = chain([3, 3, 3, 3], 0.5)
    with pytest.raises(ValueError):
        S.hybrid_steps(pats, 2, 2)
