"""Oracle: CSR transposed Jacobians and sparse products (test infrastructure).

CSR follows the SciPy convention (indptr, indices, data).  Rows are
the *input* space of the operator, columns its output space (a transposed
Jacobian J^T = (dx_i/dx_{i-1})^T).  Flat indices are channel-major then
row-major: (c*h + y)*w + x.

Contents
  * Algs. 2-4  conv 3x3/pad-1 J^T as printed, with readings 15-16
  * conv_tjac_exact        the exact guaranteed-zero stencil pattern (reading 17)
  * Algs. 5-7  ReLU J^T
  * Algs. 8-10 max-pool J^T (input-dependent pattern) and the
                           window ('guaranteed') pattern with 0/1 data (reading 18)
  * spmv, plan_product / execute_plan (symbolic then numeric),
    spgemm = execute_plan(plan_product(...)).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

D = np.float64


@dataclass
class CSR:
    rows: int
    cols: int
    indptr: np.ndarray      # int64 [rows+1]
    indices: np.ndarray     # int64 [nnz]
    data: np.ndarray | None = None   # [nnz] or [B, nnz]

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def pattern(self) -> "CSR":
        return CSR(self.rows, self.cols, self.indptr, self.indices, None)


def check(m: CSR) -> None:
    """Structural invariants."""
    ip, ix = m.indptr, m.indices
    assert len(ip) == m.rows + 1 and ip[0] == 0 and ip[-1] == len(ix)
    assert np.all(np.diff(ip) >= 0)
    if len(ix):
        assert ix.min() >= 0 and ix.max() < m.cols
        rid = np.repeat(np.arange(m.rows), np.diff(ip))
        same = rid[1:] == rid[:-1]
        assert np.all(ix[1:][same] > ix[:-1][same]), "indices not strictly increasing in a row"
    if m.data is not None:
        assert m.data.shape[-1] == len(ix)


def row_ids(m: CSR) -> np.ndarray:
    return np.repeat(np.arange(m.rows, dtype=np.int64), np.diff(m.indptr))


def to_dense(m: CSR, b: int | None = None) -> np.ndarray:
    A = np.zeros((m.rows, m.cols), D)
    data = m.data if b is None or m.data.ndim == 1 else m.data[b]
    A[row_ids(m), m.indices] = data
    return A


def from_dense(A: np.ndarray, keep: np.ndarray | None = None) -> CSR:
    """CSR of A; `keep` (bool mask) forces structural entries (explicit zeros)."""
    mask = (A != 0) if keep is None else keep
    r, c = np.nonzero(mask)
    ip = np.zeros(A.shape[0] + 1, np.int64)
    np.add.at(ip, r + 1, 1)
    return CSR(A.shape[0], A.shape[1], np.cumsum(ip), c.astype(np.int64), A[r, c].astype(D))


# ---------------------------------------------------------------------------
# products
# ---------------------------------------------------------------------------

def spmv(m: CSR, v: np.ndarray) -> np.ndarray:
    """y[i] = sum_{p in row i} data[p] v[indices[p]]  (eqn:backprop step).
    v: [cols] or [B, cols]; data [nnz] (shared) or [B, nnz]."""
    v = np.asarray(v, D)
    batched = v.ndim == 2
    V = v if batched else v[None]
    data = np.asarray(m.data, D)
    data = np.broadcast_to(data, (V.shape[0], m.nnz)) if data.ndim == 1 else data
    prod = data * V[:, m.indices]
    y = np.zeros((V.shape[0], m.rows), D)
    rid = row_ids(m)
    for b in range(V.shape[0]):
        y[b] = np.bincount(rid, weights=prod[b], minlength=m.rows)
    return y if batched else y[0]


@dataclass
class Plan:
    """Symbolic product of two patterns: output pattern plus, for every
    output entry e, the contribution pairs (left position, right position)
    listed in contrib_ptr[e]:contrib_ptr[e+1], in ascending left position."""
    out: CSR
    contrib_ptr: np.ndarray
    left_pos: np.ndarray
    right_pos: np.ndarray


def plan_product(left: CSR, right: CSR) -> Plan:
    """Structural product left @ right: every (i, k) of left meets every (k, j) of
    right.  Done once, ahead of the numeric phase."""
    if left.cols != right.rows:
        raise ValueError("incompatible shapes")
    rlen = np.diff(right.indptr)
    cnt = rlen[left.indices]                                   # pairs per left entry
    lp = np.repeat(np.arange(left.nnz, dtype=np.int64), cnt)
    first = np.repeat(right.indptr[left.indices], cnt)
    offs = np.arange(len(lp), dtype=np.int64) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    rp = first + offs
    key = row_ids(left)[lp] * right.cols + right.indices[rp]
    order = np.lexsort((lp, key))                              # by key, then left position
    key, lp, rp = key[order], lp[order], rp[order]
    uk, start = np.unique(key, return_index=True)
    orow = uk // right.cols
    ocol = uk % right.cols
    ip = np.zeros(left.rows + 1, np.int64)
    np.add.at(ip, orow + 1, 1)
    out = CSR(left.rows, right.cols, np.cumsum(ip), ocol.astype(np.int64), None)
    cptr = np.append(start, len(key)).astype(np.int64)
    return Plan(out, cptr, lp, rp)


def execute_plan(plan: Plan, left_data, right_data) -> np.ndarray:
    """Numeric phase: out[e] = sum over plan contributions of left*right, in the
    plan's order.  Data may be [nnz] or [B, nnz] (broadcast)."""
    L, R = np.asarray(left_data, D), np.asarray(right_data, D)
    prod = L[..., plan.left_pos] * R[..., plan.right_pos]
    seg = np.repeat(np.arange(plan.out.nnz), np.diff(plan.contrib_ptr))
    if prod.ndim == 1:
        return np.bincount(seg, weights=prod, minlength=plan.out.nnz)
    return np.stack([np.bincount(seg, weights=p, minlength=plan.out.nnz) for p in prod])


def spgemm(a: CSR, b: CSR) -> CSR:
    """a @ b keeping the structural product pattern (explicit zeros retained)."""
    plan = plan_product(a, b)
    out = plan.out
    return CSR(out.rows, out.cols, out.indptr, out.indices, execute_plan(plan, a.data, b.data))


# ---------------------------------------------------------------------------
# Builders
# ---------------------------------------------------------------------------

def conv_tjac_algs(ci: int, co: int, h: int, w: int, weights) -> CSR:
    """Algs. 2-4 as printed, for h, w >= 3.

    Alg. 2 indptr (three-case formula; reading 15 — the boundary cases agree),
    Alg. 3 indices (3x3 neighbourhood, `mod (c_o h w)`, rows sorted),
    Alg. 4 data (flatten(weights[:, m, range, ::-1])).  Reading 16 for the
    unexpanded 'Fix corner cases': each data value stays attached to the
    index it was generated for (the permutation applied by sorted() is applied to
    data too) and entries that are not true 3x3 neighbours (left/right wrap) get
    data 0 — explicit zeros in the padded allocation 3w(3h-2) c_i c_o."""
    W = np.asarray(weights, D)
    hw = h * w
    n_rows = ci * hw
    ip = np.empty(n_rows + 1, np.int64)
    blk = co * (3 * w * (3 * h - 2))
    for i in range(n_rows + 1):                       # Alg. 2
        a, b = divmod(i, hw)
        if b <= w:
            ip[i] = a * blk + 6 * co * b
        elif b <= w * (h - 1):
            ip[i] = a * blk + 6 * co * w + 9 * co * (b - w)
        else:
            ip[i] = a * blk + 6 * co * w + 9 * co * (w * (h - 2)) + 6 * co * (b - w * (h - 1))
    nnz = ip[-1]
    idx = np.empty(nnz, np.int64)
    dat = np.empty(nnz, D)
    off = np.array([-1, 0, 1])
    for i in range(n_rows):                           # Algs. 3 and 4
        r = i % hw
        m = i // hw
        base = np.empty(9 * co, np.int64)
        for j in range(co):
            for k in range(3):
                base[9 * j + 3 * k: 9 * j + 3 * (k + 1)] = (off + (j * h + k - 1) * w + r) % (co * hw)
        if r < w or r >= w * (h - 1):
            left, right = (3, 9) if r < w else (0, 6)
            row = np.concatenate([base[9 * j + left: 9 * j + right] for j in range(co)])
        else:
            row = base
        if r < w:
            rng_rows = [1, 0]
        elif r >= w * (h - 1):
            rng_rows = [2, 1]
        else:
            rng_rows = [2, 1, 0]
        data = W[:, m][:, rng_rows][:, :, ::-1].reshape(-1)
        order = np.argsort(row, kind="stable")
        row, data = row[order], data[order]
        # fix corner cases: zero every entry that is not a genuine neighbour
        yi, xi = divmod(r, w)
        oc, opix = np.divmod(row, hw)
        yo, xo = np.divmod(opix, w)
        ok = (np.abs(yo - yi) <= 1) & (np.abs(xo - xi) <= 1)
        data = np.where(ok, data, 0.0)
        idx[ip[i]:ip[i + 1]] = row
        dat[ip[i]:ip[i + 1]] = data
    return CSR(n_rows, co * hw, ip, idx, dat)


def conv_tjac_exact(ci: int, co: int, h: int, w: int, weights=None,
                    drop_zero_weights: bool = False) -> CSR:
    """Exact guaranteed-zero pattern of a 3x3, pad-1, stride-1 conv J^T:
    entry (input (c_i, y_i, x_i), output (c_o, y_o, x_o)) exists iff
    |y_o - y_i| <= 1 and |x_o - x_i| <= 1, value W[c_o, c_i, y_i-y_o+1, x_i-x_o+1]
    (out = cross-correlation).  nnz = c_i c_o (3h-2)(3w-2) for h, w >= 2
    (reading 17).  With drop_zero_weights the pruned filter taps are removed
    from the pattern (they are zero for the whole retraining)."""
    CO = np.arange(co).reshape(1, 1, 1, co, 1, 1)
    YI = np.arange(h).reshape(1, h, 1, 1, 1, 1)
    XI = np.arange(w).reshape(1, 1, w, 1, 1, 1)
    OY = np.arange(-1, 2).reshape(1, 1, 1, 1, 3, 1)
    OX = np.arange(-1, 2).reshape(1, 1, 1, 1, 1, 3)
    shape = (ci, h, w, co, 3, 3)
    valid = np.broadcast_to((YI + OY >= 0) & (YI + OY < h) & (XI + OX >= 0) & (XI + OX < w), shape)
    col = np.broadcast_to(CO * h * w + (YI + OY) * w + (XI + OX), shape)
    vals = None
    if weights is not None:
        Wt = np.asarray(weights, D)                                  # [co, ci, 3, 3]
        # value at (ci, ., ., co, oy, ox) = W[co, ci, 1-oy, 1-ox]
        vals = Wt[:, :, ::-1, ::-1].transpose(1, 0, 2, 3).reshape(ci, 1, 1, co, 3, 3)
        vals = np.broadcast_to(vals, shape)
        if drop_zero_weights:
            valid = valid & (vals != 0)
    keep = valid.reshape(ci * h * w, co * 9)
    ip = np.zeros(ci * h * w + 1, np.int64)
    ip[1:] = np.cumsum(keep.sum(axis=1))
    idx = col.reshape(ci * h * w, co * 9)[keep].astype(np.int64)
    data = None if vals is None else vals.reshape(ci * h * w, co * 9)[keep].astype(D)
    return CSR(ci * h * w, co * h * w, ip, idx, data)


def relu_tjac(x) -> CSR:
    """Algs. 5-7: indptr[i] = i, indices[i] = i, data[i] = [x[i] > 0]."""
    x = np.asarray(x).reshape(-1)
    d = x.size
    return CSR(d, d, np.arange(d + 1, dtype=np.int64), np.arange(d, dtype=np.int64),
               (x > 0).astype(D))


def maxpool_tjac(pool_indices, c: int, h: int, w: int) -> CSR:
    """Algs. 8-10: window = stride = 2; pool_indices[c, yo, xo] is the
    flat index within the c-th input plane of the pooled element (torch
    max_pool2d return_indices).  One unit entry per output column."""
    pidx = np.asarray(pool_indices)
    ho, wo = pidx.shape[1], pidx.shape[2]
    mapping = np.full(c * h * w, -1, np.int64)
    for cc in range(c):                                   # Alg. 8 (parallel part)
        for yy in range(ho):
            for xx in range(wo):
                i = cc * h * w + int(pidx[cc, yy, xx])
                j = (cc * ho + yy) * wo + xx
                mapping[i] = j
    ip = np.empty(c * h * w + 1, np.int64)
    ptr = 0
    for i in range(c * h * w):                            # Alg. 8 (serial prefix)
        ip[i] = ptr
        if mapping[i] != -1:
            ptr += 1
    ip[-1] = ptr
    idx = mapping[mapping != -1]                           # Alg. 9
    return CSR(c * h * w, c * ho * wo, ip, idx.astype(np.int64), np.ones(ptr, D))   # Alg. 10


def maxpool_window_tjac(pool_indices, c: int, h: int, w: int) -> CSR:
    """Guaranteed-zero (window) pattern of a 2x2/stride-2 max-pool J^T: every
    input pixel has exactly one structural entry (its window's output) with data
    1 if it is the pooled element, else 0 (reading 18).  Table 1's max-pool
    sparsity 1 - h_f w_f/(c_i h_i w_i) counts this pattern."""
    pidx = np.asarray(pool_indices)
    ho, wo = h // 2, w // 2
    rows = np.arange(c * h * w)
    cc, rem = np.divmod(rows, h * w)
    yy, xx = np.divmod(rem, w)
    col = (cc * ho + yy // 2) * wo + xx // 2
    pooled = pidx[cc, yy // 2, xx // 2] == rem
    return CSR(c * h * w, c * ho * wo, np.arange(c * h * w + 1, dtype=np.int64),
               col.astype(np.int64), pooled.astype(D))
