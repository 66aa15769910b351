"""Dev aid: numpy emulation of candidate exact-integer (int8-slice) tensor-core
schemes for the level-0 fold chain c <- W^T (d o c), against fp64 and an fp32
FFMA-like baseline, on the norm-preserving family (SURVEY reading 12).

Integer slice products are exact in float64 (|partial sums| < 2^53); the fp32
epilogue is emulated with numpy float32 roundings in the kernel's order.

    python scripts/ozaki_sim.py [T] [H] [nchains]
"""
import sys

import numpy as np


def digits_balanced(Xint, nd):
    """balanced base-256 digits of int64 array Xint, most significant first"""
    out = []
    r = Xint.copy()
    for _ in range(nd - 1):
        d = ((r + 128) & 255) - 128
        out.append(d)
        r = (r - d) >> 8
    out.append(r)
    return out[::-1]


def run(T, H, nch, xd=3, wd=4, rmax=3, scale="exact", seed=0, wbits=None):
    wbits = 8 * wd - 1 if wbits is None else wbits
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((H, H)))
    cc = 1.0 / (1.0 - 0.01**2 / 3.0)
    W = (cc * Q).astype(np.float32)
    h = rng.uniform(-0.01, 0.01, size=(T, H)).astype(np.float32)
    d = (np.float32(1) - h * h).astype(np.float32)
    c0 = rng.standard_normal((nch, H))
    # fp64 reference (rows = chains): c <- (d o c) W
    ref = c0.copy()
    W64 = W.astype(np.float64)
    d64 = d.astype(np.float64)
    # fp32 baseline
    f32 = c0.astype(np.float32)
    # integer scheme: W digits (per-matrix scale), top digit range +-127
    mW = np.abs(W64).max()
    tau = (wbits - 1) - int(np.floor(np.log2(mW)))          # max |Wint| in [2^(wbits-1), 2^wbits)
    Wint = np.rint(W64 * 2.0**tau).astype(np.int64)
    Wd = digits_balanced(Wint, wd)                           # W0 (top) .. W_{wd-1}
    wshift = 8 * (wd - 1)                                    # Wint = sum Wj 256^(wd-1-j)
    Wdf = [w.astype(np.float64) for w in Wd]
    cI = c0.astype(np.float32)
    E = np.zeros(nch)                                        # c_true = cI * 2^E
    m_prev = None
    for t in range(T):
        ref = (d64[t] * ref) @ W64
        xf = (d[t] * f32).astype(np.float32).astype(np.float64)
        acc = np.zeros((nch, H), np.float32)
        for k in range(H):                                   # sequential FMA over k
            acc = (acc.astype(np.float64) + xf[:, k:k + 1] * W64[k][None, :]).astype(np.float32)
        f32 = acc
        y = (d[t] * cI).astype(np.float32)                   # FMUL
        if scale == "exact":
            m = np.abs(y).max(axis=1)
        else:                                                # bound from previous step (loose)
            m = np.abs(y).max(axis=1) * 8.0
        m = np.where(m > 0, m, 1.0)
        sig = (8 * xd - 3) - np.floor(np.log2(m)).astype(np.int64)   # max |X| in [2^(8xd-3), 2^(8xd-2))
        X = np.rint(y.astype(np.float64) * np.ldexp(1.0, sig)[:, None]).astype(np.int64)
        assert np.abs(X).max() < 2 ** (8 * xd - 2)
        Xd = digits_balanced(X, xd)
        Xdf = [x.astype(np.float64) for x in Xd]
        R = [np.zeros((nch, H)) for _ in range(rmax + 1)]
        for i in range(xd):
            for j in range(wd):
                if i + j <= rmax:
                    R[i + j] += Xdf[i] @ Wdf[j]
        mr = max(np.abs(r).max() for r in R)
        if mr >= 2**22 and t == 0: print("  (region exceeds 2^22:", mr, ")")
        # fp32 Horner with magic-number integer roundings for the lower regions
        v = R[rmax]
        for r in range(rmax - 1, 0, -1):
            v = np.rint(R[r] + v / 256.0)                    # ulp-1 rounding (biased magic)
        cI = (R[0] + v / 256.0).astype(np.float32)           # one RN rounding (FFMA)
        # true scale: X = y 2^sig; X.W = 256^(xd-1) 256^(wd-1) sum R_r 256^-r
        E = E + 0  # track exponent exactly in float64 instead of int bookkeeping
        scale_c = np.ldexp(1.0, 8 * (xd - 1) + wshift - tau) / np.ldexp(1.0, sig)
        # renormalise the fp32 state: cI holds c_true / 2^E
        E = E + np.log2(scale_c)
        # keep cI as is (fp32) ; fold scale in E
    ctrue = cI.astype(np.float64) * np.exp2(E)[:, None]
    err_int = np.abs(ctrue - ref).max() / np.abs(ref).max()
    err_f32 = np.abs(f32.astype(np.float64) - ref).max() / np.abs(ref).max()
    return err_int, err_f32


if __name__ == "__main__":
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    nch = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    for (xd, wd, rmax, sc) in [(3, 4, 3, "exact"), (3, 3, 2, "exact"), (3, 4, 3, "bound"), (3, 4, 2, "exact"),
                               (4, 4, 3, "exact")]:
        ei, ef = run(T, H, nch, xd, wd, rmax, sc)
        print(f"T={T} H={H} x{xd} w{wd} r<={rmax} {sc:5s}: int-scheme {ei:.3e}   fp32 matmul {ef:.3e}", flush=True)
