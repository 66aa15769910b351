"""Oracle: the scan formulation of BP, executed literally (test infrastructure).

Scan array (eqn:scan_input) for a chain of T steps, in *scan order*:

    a = [seed, J_{T-1}^T, J_{T-2}^T, ..., J_0^T]          (n = T, n+1 slots)

so slot k >= 1 holds J_{T-k}^T.  The exclusive scan with the
operator A <> B = B A yields [I, grad_h[T-1], ..., grad_h[0]]
(Alg. 1 "Ensure"); the last slot J_0^T only enters the inclusive total
(reading 3).  Elements are batched over B samples: a vector is [B,H], a matrix
[B,H,H]; the identity is symbolic and never materialised.
"""
from __future__ import annotations

from collections import Counter
from dataclasses import dataclass

import numpy as np

from . import csr

D = np.float64


@dataclass
class El:
    kind: str                      # 'I' (symbolic identity) | 'v' | 'm' | 's' (CSR)
    val: np.ndarray | None = None


IDENT = El("I")


def diamond(A: El, B: El, stats: Counter | None = None) -> El:
    """A <> B = B A.  A: identity, vector or matrix; B: identity or matrix.
    The identity short-circuits (no multiplication; 'logical data movement')."""
    if A.kind == "I":
        if stats is not None:
            stats["copy"] += 1
        return B
    if B.kind == "I":
        if stats is not None:
            stats["copy"] += 1
        return A
    if B.kind not in ("m", "s"):
        raise ValueError("right operand of <> must be a matrix")
    if A.kind == "v":
        if stats is not None:
            stats["mv"] += 1
        if B.kind == "s":                                  # CSR J^T times vector
            return El("v", csr.spmv(B.val, A.val))
        return El("v", np.einsum("bik,bk->bi", B.val, A.val))
    if stats is not None:
        stats["mm"] += 1
    if B.kind == "s" and A.kind == "s":                    # CSR SpGEMM
        return El("s", csr.spgemm(B.val, A.val))
    if A.kind == "s" or B.kind == "s":
        raise ValueError("mixed dense/CSR matrix product is not used")
    return El("m", np.einsum("bij,bjk->bik", B.val, A.val))


def scan_array(seed, JT_time):
    """Build eqn:scan_input from seed [B,H] and JT_time[t] = J_t^T ([T,B,H,H])."""
    T = JT_time.shape[0]
    a = [El("v", np.asarray(seed, D))]
    for k in range(1, T + 1):
        a.append(El("m", np.asarray(JT_time[T - k], D)))
    return a


def linear_scan(a, stats: Counter | None = None):
    """Serial exclusive scan: out[0] = I, out[k] = a[0] <> ... <> a[k-1]."""
    out, acc = [IDENT], IDENT
    for k in range(len(a) - 1):
        acc = diamond(acc, a[k], stats)
        out.append(acc)
    return out


def num_levels(n: int) -> int:
    """L = ceil(log2(n+1)) for n >= 1 (reading 4)."""
    return int(n).bit_length()


def blelloch(a, stats: Counter | None = None, trace: list | None = None,
             modified: bool = True, phase_stats: dict | None = None):
    """Alg. 1 executed literally, in place on a copy of `a`.

    Up-sweep   d = 0 .. L-2:  a[r] <- a[l] <> a[r]
    a[n] <- I
    Down-sweep d = L-1 .. 0:  T <- a[l]; a[l] <- a[r]; a[r] <- a[r] <> T
    with (l, r) = (i + 2^d - 1, min(i + 2^{d+1} - 1, n)), i = 0 .. n-2^d step 2^{d+1}
    (inclusive bounds, reading 4).  `modified=False` runs the textbook
    down-sweep a[r] <- T <> a[r] (the negative test of P:135 / S:256).
    `trace` receives one (phase, d, [(l, r), ...]) record per level."""
    a = list(a)
    n = len(a) - 1
    L = num_levels(n)
    for d in range(0, L - 1):
        pairs = [(i + 2 ** d - 1, min(i + 2 ** (d + 1) - 1, n))
                 for i in range(0, n - 2 ** d + 1, 2 ** (d + 1))]
        _assert_disjoint(pairs)
        for l, r in pairs:
            if phase_stats is not None:
                _tally(phase_stats["up"], a[l], a[r])
            a[r] = diamond(a[l], a[r], stats)
        if trace is not None:
            trace.append(("up", d, pairs))
    a[n] = IDENT
    for d in range(L - 1, -1, -1):
        pairs = [(i + 2 ** d - 1, min(i + 2 ** (d + 1) - 1, n))
                 for i in range(0, n - 2 ** d + 1, 2 ** (d + 1))]
        _assert_disjoint(pairs)
        for l, r in pairs:
            T = a[l]
            a[l] = a[r]
            if phase_stats is not None:
                _tally(phase_stats["down"], a[l], T)
            a[r] = diamond(a[r], T, stats) if modified else diamond(T, a[r], stats)
        if trace is not None:
            trace.append(("down", d, pairs))
    return a


def _tally(c: Counter, A: El, B: El) -> None:
    """Classify one <> application A <> B by operand kinds (for phase counts)."""
    if A.kind == "I" or B.kind == "I":
        c["copy"] += 1
    elif A.kind == "v":
        c["mv"] += 1
    else:
        c["mm"] += 1


def _assert_disjoint(pairs):
    seen = set()
    for l, r in pairs:
        assert l not in seen and r not in seen and l != r, "pairs of one level overlap"
        seen.update((l, r))


def hybrid(a, up_levels: int, down_levels: int, stats: Counter | None = None):
    """Level-balanced scan of P:472: the first `up_levels` up-sweep levels of
    Alg. 1 (d = 0..u-1), a serial 'bridge' that folds the 2^u-block aggregates
    left to right and deposits the exclusive prefix of every 2^dl-block at that
    block's right end, then the last `down_levels` down-sweep levels
    (d = dl-1..0).  Valid for dl in {u, u+1} (reading 19); (0, 0) is the linear
    scan and (L-1, L) is Alg. 1 (the bridge then reduces to a[n] <- I)."""
    a = list(a)
    n = len(a) - 1
    u, dl = up_levels, down_levels
    L = num_levels(n)
    if not (0 <= u <= max(L - 1, 0) and dl in (u, u + 1) and dl <= L):
        raise ValueError("need 0 <= up_levels <= L-1, down_levels in {u, u+1}, down_levels <= L")
    for d in range(0, u):
        for i in range(0, n - 2 ** d + 1, 2 ** (d + 1)):
            l, r = i + 2 ** d - 1, min(i + 2 ** (d + 1) - 1, n)
            a[r] = diamond(a[l], a[r], stats)
    # bridge: serial fold over the 2^u-block aggregates
    bs = 2 ** u
    last = (n // 2 ** dl) * 2 ** dl                # start of the last 2^dl-block
    P, deposits = IDENT, []
    for s in range(0, last + 1, bs):
        if s % (2 ** dl) == 0:
            deposits.append((min(s + 2 ** dl - 1, n), P))
        if s + bs <= last:                          # fold only what a deposit needs
            P = diamond(P, a[min(s + bs - 1, n)], stats)
    for pos, val in deposits:
        a[pos] = val
    for d in range(dl - 1, -1, -1):
        for i in range(0, n - 2 ** d + 1, 2 ** (d + 1)):
            l, r = i + 2 ** d - 1, min(i + 2 ** (d + 1) - 1, n)
            T = a[l]
            a[l] = a[r]
            a[r] = diamond(a[r], T, stats)
    return a


def grads_from_scan(out):
    """Map the exclusive-scan output [I, g_{T-1}, ..., g_0] to grad_h[t] ([T,B,H])."""
    T = len(out) - 1
    return np.stack([out[T - t].val for t in range(T)])


# ---------------------------------------------------------------------------
# Multi-GPU protocol emulation (contiguous time shards)
# ---------------------------------------------------------------------------

def shard_bounds(T: int, G: int):
    """Contiguous shards in time order: rank r owns t in [lo_r, hi_r) with the
    remainder spread over the first ranks."""
    base, rem = divmod(T, G)
    out, lo = [], 0
    for r in range(G):
        sz = base + (1 if r < rem else 0)
        out.append((lo, lo + sz))
        lo += sz
    return out


def shard_aggregate(JT_time, lo, hi, seed=None):
    """Aggregate of a shard: the product J_lo^T J_{lo+1}^T ... J_{hi-1}^T (plain
    sequential product), applied to `seed` when the shard holds t = T-1
    (its aggregate is then the vector grad_h[lo-1])."""
    JT = np.asarray(JT_time[lo:hi], D)
    if seed is not None:
        v = np.asarray(seed, D)
        for t in range(hi - lo - 1, -1, -1):
            v = np.einsum("bik,bk->bi", JT[t], v)
        return El("v", v)
    P = JT[hi - lo - 1].copy()
    for t in range(hi - lo - 2, -1, -1):
        P = np.einsum("bij,bjk->bik", JT[t], P)
    return El("m", P)


def shard_carries(aggs):
    """carry[r] = dl/dh at the shard's last step: carry[G-1] = seed (handled by
    the caller), carry[r] = M_{r+1} ... M_{G-2} V_{G-1} for r < G-1."""
    G = len(aggs)
    carries = [None] * G
    if G >= 2:
        v = aggs[G - 1].val
        carries[G - 2] = v
        for r in range(G - 3, -1, -1):
            v = np.einsum("bik,bk->bi", aggs[r + 1].val, v)
            carries[r] = v
    return carries


def shard_local_grads(JT_time, lo, hi, carry):
    """grad_h[t] for t in [lo, hi) given carry = grad_h[hi-1]."""
    v = np.asarray(carry, D).copy()
    out = np.empty((hi - lo,) + v.shape, D)
    for t in range(hi - 1, lo - 1, -1):
        out[t - lo] = v
        v = np.einsum("bik,bk->bi", np.asarray(JT_time[t], D), v)
    return out, v


def hybrid_steps(patterns, up_levels: int, down_levels: int):
    """Static FLOP analysis of the hybrid schedule (fig:prune_symbolic, P:467,
    P:474) over a CSR chain given by its patterns only.

    `patterns[k]` = csr.CSR pattern of J_{k+1}^T in time order (data unused).
    The scan array is [seed, J_n^T, ..., J_1^T] (reading 3); the schedule is
    `hybrid` above step by step, each <> application recorded as one op:
      mm  a[r] <- a[l] <> a[r] = a[r] a[l] with both matrices:
          flops = 2 x the contribution pairs of the structural product
          (csr.plan_product), dense_flops = 2 m k n;
      mv  any product with a vector: flops = 2 nnz(matrix), dense = 2 m n.
    Identities are symbolic (no op).  Then the inclusive extra
    J_1^T dl/dx_1 (phase 'extra') and the BP baseline's n gradient operators
    J_n^T .. J_1^T (phase 'bp', level k).  critical (reading 23): the costliest
    op of each up/down level (first on ties); every bridge/extra/bp op."""
    n = len(patterns)
    u, dl = up_levels, down_levels
    L = num_levels(n)
    if not (0 <= u <= max(L - 1, 0) and dl in (u, u + 1) and dl <= L):
        raise ValueError("need 0 <= up_levels <= L-1, down_levels in {u, u+1}, down_levels <= L")
    VEC, ID = "v", "I"
    a = [VEC] + [patterns[n - s] for s in range(1, n + 1)]      # slot s >= 1: J_{n-s+1}^T
    steps = []

    def op(phase, level, left, right):
        """left <> right = right . left; returns the result (VEC or a pattern)."""
        if left is ID:
            return right
        if right is ID:
            return left
        if left is VEC:
            steps.append(dict(kind="mv", phase=phase, level=level, flops=2 * right.nnz,
                              dense_flops=2 * right.rows * right.cols))
            return VEC
        pl = csr.plan_product(right, left)
        steps.append(dict(kind="mm", phase=phase, level=level, flops=2 * len(pl.left_pos),
                          dense_flops=2 * right.rows * right.cols * left.cols))
        return pl.out

    for d in range(0, u):
        for i in range(0, n - 2 ** d + 1, 2 ** (d + 1)):
            l, r = i + 2 ** d - 1, min(i + 2 ** (d + 1) - 1, n)
            a[r] = op("up", d, a[l], a[r])
    bs, D = 2 ** u, 2 ** dl
    last = (n // D) * D
    P, deposits = ID, []
    for s in range(0, last + 1, bs):
        if s % D == 0:
            deposits.append((min(s + D - 1, n), P))
        if s + bs <= last:
            P = op("bridge", s // bs, P, a[min(s + bs - 1, n)])
    for pos, val in deposits:
        a[pos] = val
    for d in range(dl - 1, -1, -1):
        for i in range(0, n - 2 ** d + 1, 2 ** (d + 1)):
            l, r = i + 2 ** d - 1, min(i + 2 ** (d + 1) - 1, n)
            T = a[l]
            a[l] = a[r]
            a[r] = op("down", d, a[r], T)
    assert all(x is VEC for x in a[1:]), "every output slot must be a vector"
    op("extra", 0, VEC, patterns[0])
    for st in steps:
        st["critical"] = st["phase"] in ("bridge", "extra")
    for ph in ("up", "down"):
        for lv in {st["level"] for st in steps if st["phase"] == ph}:
            grp = [st for st in steps if st["phase"] == ph and st["level"] == lv]
            max(grp, key=lambda st: st["flops"])["critical"] = True     # max() keeps the first on ties
    for k in range(n, 0, -1):
        m = patterns[k - 1]
        steps.append(dict(kind="mv", phase="bp", level=k, flops=2 * m.nnz, dense_flops=2 * m.rows * m.cols,
                          critical=True))
    return steps
