"""Pins for oracle/scan.py: Alg. 1 structure, exactness on integer
non-commutative chains, hybrid degenerate cases, the down-sweep reversal
(P:135), shard-protocol emulation, and the integer families the GPU must match
bit-exactly."""
import json
import os
from collections import Counter

import numpy as np
import pytest

import bppsa_workloads as W
from oracle import bp, scan as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _int_chain(n, B=2, H=3, seed=0, vec_head=True):
    """Exact non-commutative integer chains: dense {-1,0,1} matrices for short
    chains; for long ones the non-expansive column-function family (values stay
    small integers under any association)."""
    rng = np.random.default_rng(seed)
    head = (S.El("v", rng.integers(-2, 3, (B, H)).astype(float)) if vec_head
            else S.El("m", rng.integers(-2, 3, (B, H, H)).astype(float)))
    if n <= 40:
        mats = rng.integers(-1, 2, (n, B, H, H)).astype(float)
    else:
        mats = W.int_dense_family(n, B, H, seed=seed, n_copy=8, p_merge=0.3)["JT"].astype(float)
    return [head] + [S.El("m", m) for m in mats]


@pytest.mark.parametrize("n", list(range(1, 70)) + [127, 128, 129, 255, 1000, 1023, 1024])
def test_alg1_equals_exclusive_scan_exactly(n):
    """Alg. 1 Ensure clause on integer matrices (exact in fp64), plus the
    exact operation and level counts of Appendix A / S:253-254."""
    a = _int_chain(n, seed=n)
    lin = S.linear_scan(a)
    ph = {"up": Counter(), "down": Counter()}
    trace = []
    out = S.blelloch(a, trace=trace, phase_stats=ph)
    assert out[0].kind == "I"
    for k in range(1, n + 1):
        assert out[k].kind == "v" and np.array_equal(out[k].val, lin[k].val)
    L = S.num_levels(n)
    assert L == int(np.ceil(np.log2(n + 1)))
    assert len(trace) == 2 * L - 1                              # levels
    assert sum(1 for t in trace if t[0] == "up") == L - 1
    assert ph["up"]["mm"] == n - L and ph["up"]["mv"] == L - 1 and ph["up"]["copy"] == 0
    # "Only the up-sweep phase contains matrix-matrix multiplications"
    assert ph["down"]["mm"] == 0 and ph["down"]["mv"] == n - L and ph["down"]["copy"] == L
    total = sum(ph["up"].values()) + sum(ph["down"].values())
    assert total == 2 * n - 1 <= 2 * (n + 1)                     # W = Theta(n)


def test_alg1_n7_golden():
    g = GOLD["alg1_n7"]
    trace = []
    st = Counter()
    S.blelloch(_int_chain(g["n"]), stats=st, trace=trace)
    assert sum(1 for t in trace if t[0] == "up") == g["up_levels"]
    assert sum(1 for t in trace if t[0] == "down") == g["down_levels"]
    assert sum(st.values()) == g["diamond_ops"]


def test_unmodified_down_sweep_is_wrong_for_n_ge_3():
    """P:135 / S:256: without the operand reversal of line 13 the result differs
    from the exclusive scan for every n >= 3 (and coincides for n = 1, 2)."""
    for n in range(1, 65):
        a = _int_chain(n, seed=100 + n, vec_head=False)
        lin = S.linear_scan(a)
        neg = S.blelloch(a, modified=False)
        wrong = any(not np.array_equal(lin[k].val, neg[k].val) for k in range(1, n + 1))
        assert wrong == (n >= 3), n


def test_scalar_chain_golden():
    g = GOLD["scalar_chain"]
    vals = g["inputs"]
    a = [S.El("v", np.array([[vals[0]]], float))] + [S.El("m", np.array([[[v]]], float)) for v in vals[1:]]
    for out in (S.linear_scan(a), S.blelloch(a)):
        got = [1.0] + [float(o.val[0, 0]) for o in out[1:]]
        assert got == g["exclusive_scan"]


def test_diamond_golden_and_identity():
    g = GOLD["diamond_example"]
    A = S.El("v", np.array([g["A"]], float))
    B = S.El("m", np.array([g["B"]], float))
    assert S.diamond(A, B).val[0].tolist() == g["result"]
    assert S.diamond(A, S.IDENT) is A and S.diamond(S.IDENT, B) is B


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 20, 21, 100, 257])
def test_hybrid_all_valid_splits(n):
    """Hybrid equals the exclusive scan for every valid (u, dl); (0, 0)
    is the linear scan op-for-op and (L-1, L) reproduces Alg. 1's result."""
    a = _int_chain(n, seed=7 * n)
    lin = S.linear_scan(a)
    L = S.num_levels(n)
    for u in range(0, L):
        for dl in (u, u + 1):
            if dl > L:
                continue
            out = S.hybrid(a, u, dl)
            for k in range(1, n + 1):
                assert np.array_equal(out[k].val, lin[k].val), (u, dl, k)
    s_lin, s_h = Counter(), Counter()
    S.linear_scan(a, s_lin)
    S.hybrid(a, 0, 0, s_h)
    assert s_lin == s_h
    s_b, s_h = Counter(), Counter()
    S.blelloch(a, s_b)
    S.hybrid(a, L - 1, L, s_h)
    assert s_b == s_h


def test_vgg_hybrid_labels():
    """P:472 on the n = 21 VGG-11 chain: up-sweep L0-L2 (u = 3), down L7-L10 (dl = 4)."""
    a = _int_chain(21, seed=11)
    lin = S.linear_scan(a)
    out = S.hybrid(a, 3, 4)
    for k in range(1, 22):
        assert np.array_equal(out[k].val, lin[k].val)


def test_linear_scan_is_sequential_bp():
    """The serial exclusive scan over eqn:scan_input performs exactly the BP
    recurrence (same operations in the same order)."""
    T, B, H = 40, 3, 5
    rng = np.random.default_rng(2)
    JT = rng.standard_normal((T, B, H, H))
    g = rng.standard_normal((B, H))
    ref, _ = bp.bp_dense(JT, g)
    out = S.linear_scan(S.scan_array(g, JT))
    assert np.array_equal(S.grads_from_scan(out), ref)
    blel = S.grads_from_scan(S.blelloch(S.scan_array(g, JT)))
    assert np.abs(blel - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("T,G", [(1, 1), (7, 2), (100, 3), (64, 8), (1000, 8), (5, 5)])
def test_shard_protocol_equals_monolithic(T, G):
    """Contiguous time shards: local aggregates, carries
    M_{r+1}...M_{G-2} V_{G-1}, local down-walk == monolithic sequential BP."""
    B, H = 2, 4
    rng = np.random.default_rng(T * 10 + G)
    JT = rng.standard_normal((T, B, H, H)) * 0.5
    g = rng.standard_normal((B, H))
    ref, ref_init = bp.bp_dense(JT, g)
    bounds = S.shard_bounds(T, G)
    assert bounds[0][0] == 0 and bounds[-1][1] == T
    assert all(bounds[r][1] == bounds[r + 1][0] for r in range(G - 1))
    aggs = [S.shard_aggregate(JT, lo, hi, g if r == G - 1 else None) for r, (lo, hi) in enumerate(bounds)]
    carries = S.shard_carries(aggs)
    carries[G - 1] = g
    got = np.concatenate([S.shard_local_grads(JT, lo, hi, carries[r])[0] for r, (lo, hi) in enumerate(bounds)])
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)
    _, init = S.shard_local_grads(JT, *bounds[0], carries[0])
    assert np.allclose(init, ref_init, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------ integer families

def test_int_dense_family_is_exact_under_any_association():
    """The column-function family: ||J^T||_1 <= 1 except n_copy matrices with
    ||.||_1 = 2, so every window product and every GEMV partial sum stays below
    2^24: chain (BP) == Alg. 1 tree exactly, all integers."""
    T, B, H = 300, 3, 20
    f = W.int_dense_family(T, B, H, seed=5, n_copy=10)
    JT, g = f["JT"].astype(np.float64), f["g"].astype(np.float64)
    colsum = np.abs(JT).sum(axis=2)               # [T,B,H] column abs sums
    assert colsum.max() <= 2 and (colsum == 2).sum() <= 10
    ref, _ = bp.bp_dense(JT, g)
    assert np.array_equal(ref, np.round(ref))
    bound = np.abs(g).sum(axis=1).max() * 2 ** 10
    assert np.abs(ref).max() <= bound < 2 ** 24
    tree = S.grads_from_scan(S.blelloch(S.scan_array(g, JT)))
    assert np.array_equal(tree, ref)
    assert (ref != 0).mean() > 0.3


def test_int_rnn_family_exact():
    T, B, H = 500, 4, 20
    f = W.int_rnn_family(T, B, H, seed=3)
    ref, _ = bp.bp_rnn(f["h"], f["W_hh"], f["g"])
    assert np.array_equal(ref, np.round(ref)) and np.abs(ref).max() <= 8
    JT = np.stack([bp.rnn_jt(f["h"][t], f["W_hh"]) for t in range(T)])
    tree = S.grads_from_scan(S.blelloch(S.scan_array(f["g"], JT)))
    assert np.array_equal(tree, ref)
    assert (ref != 0).mean() > 0.5


def test_gru_zero_family_powers_of_two():
    """P3(iii): J^T = 0.5 I -> grad_h[t] = 0.5^{T-1-t} g exactly."""
    T, B, H = 100, 2, 20
    f = W.gru_zero_family(T, B, H, seed=1)
    ref, _ = bp.bp_gru(f["tape"], f["W_hh3"], f["g"])
    for t in range(T):
        assert np.array_equal(ref[t], f["g"] * 0.5 ** (T - 1 - t))


def test_gru_int_family_column_function():
    T, B, H = 200, 2, 20
    f = W.gru_int_family(T, B, H, seed=2)
    for t in (0, 57, 199):
        JT = bp.gru_jt(*(f["tape"][k][t] for k in ("h_prev", "r", "z", "n", "M")), f["W_hh3"])
        assert set(np.unique(JT)) <= {-1.0, 0.0, 1.0}
        assert (np.abs(JT).sum(axis=1) <= 1).all()      # each column of J^T: <= 1 nonzero
    ref, _ = bp.bp_gru(f["tape"], f["W_hh3"], f["g"])
    assert np.array_equal(ref, np.round(ref))
