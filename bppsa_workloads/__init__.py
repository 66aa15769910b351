"""Seeded synthetic inputs for BPPSA — shared by the oracle side and the CUDA side.

This module holds NONE of BPPSA's arithmetic (no Jacobian products, no scan,
no back-propagation).  It only draws random numbers and runs the *forward*
model that produces the saved activations the backward pass consumes, the way
the paper's experiments do (cuDNN forward), here in fp32 numpy on
the host so that both sides see byte-identical inputs:

* bitstream classification data, x_t ~ Bernoulli(0.05 + 0.1 c)
* tanh-RNN forward h_t = tanh(W_ih x_t + b_ih + W_hh h_{t-1} + b_hh)
* GRU forward with gates r, z, n and M = W_hn h_{t-1} + b_hn
* IRMAS-shaped MFCC-like features (F x C from Table 3)
* the softmax/cross-entropy head gradient that seeds the scan (a0)
* integer-valued and norm-preserving families used by the parity tests
* VGG-11 conv-stack weights (97 % magnitude-pruned), images, and the forward
  that yields ReLU masks / max-pool indices for the CSR variant

Every generator takes an explicit seed and uses numpy's PCG64 (default_rng).
The recipes are listed in DESIGN.md ("Input recipes").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32


def _rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


# --------------------------------------------------------------------------
# tanh RNN, bitstream task
# --------------------------------------------------------------------------

def bitstreams(T: int, B: int, seed: int, classes: int = 10):
    """x[t, b, 0] ~ Bernoulli(0.05 + 0.1 c_b), c_b ~ U{0..9}."""
    g = _rng(seed)
    labels = g.integers(0, classes, size=B)
    p = 0.05 + 0.1 * labels.astype(np.float64)
    x = (g.random((T, B)) < p[None, :]).astype(F32)[:, :, None]
    return x, labels.astype(np.int64)


def rnn_params(H: int, I: int = 1, classes: int = 10, seed: int = 0):
    """torch nn.RNN / nn.Linear default init: U(-1/sqrt(H), 1/sqrt(H))."""
    g = _rng(seed)
    k = 1.0 / math.sqrt(H)
    u = lambda *s: g.uniform(-k, k, size=s).astype(F32)
    return dict(W_ih=u(H, I), W_hh=u(H, H), b_ih=u(H), b_hh=u(H),
                W_out=u(classes, H), b_out=u(classes))


def rnn_forward(x: np.ndarray, p: dict, h0: np.ndarray | None = None) -> np.ndarray:
    """fp32 forward of eqn:rnn; returns h[t] for t = 0..T-1 (time-major [T,B,H])."""
    T, B, _ = x.shape
    H = p["W_hh"].shape[0]
    h = np.zeros((B, H), F32) if h0 is None else h0.astype(F32).copy()
    out = np.empty((T, B, H), F32)
    Wih_T = np.ascontiguousarray(p["W_ih"].T)
    Whh_T = np.ascontiguousarray(p["W_hh"].T)
    bias = (p["b_ih"] + p["b_hh"]).astype(F32)
    pre_in = x @ Wih_T  # [T,B,H]; input projection has no recurrence
    for t in range(T):
        h = np.tanh(pre_in[t] + bias + h @ Whh_T)
        out[t] = h
    return out


def head_seed(h_last: np.ndarray, W_out: np.ndarray, b_out: np.ndarray,
              labels: np.ndarray) -> np.ndarray:
    """Seed a0 = dl/dh_{T-1} for mean softmax cross-entropy on h_{T-1}.

    This is the classifier head's derivative (input to the scan, not the scan).
    """
    B = h_last.shape[0]
    logits = h_last.astype(np.float64) @ W_out.T.astype(np.float64) + b_out
    logits -= logits.max(axis=1, keepdims=True)
    pr = np.exp(logits)
    pr /= pr.sum(axis=1, keepdims=True)
    pr[np.arange(B), labels] -= 1.0
    return (pr @ W_out.astype(np.float64) / B).astype(F32)


@dataclass
class RnnWorkload:
    x: np.ndarray          # [T,B,I]
    labels: np.ndarray     # [B]
    params: dict
    h: np.ndarray          # [T,B,H]
    g: np.ndarray          # [B,H]  seed = dl/dh_{T-1}
    h_init: np.ndarray | None = None

    @property
    def W_hh(self):
        return self.params["W_hh"]


def rnn_workload(T: int, B: int, H: int, seed: int = 0, I: int = 1) -> RnnWorkload:
    """Configs 1, 2, 4 (realistic family): bitstreams + torch-default init + fp32 forward."""
    x, labels = bitstreams(T, B, seed)
    p = rnn_params(H, I, 10, seed + 1)
    h = rnn_forward(x, p)
    g = head_seed(h[-1], p["W_out"], p["b_out"], labels)
    return RnnWorkload(x, labels, p, h, g)


def per_step_seeds(w: RnnWorkload, seed: int = 0) -> np.ndarray:
    """Per-step losses: a label y_t ~ U{0..9} per step and the
    same head on every h_t; e[t] = dl_t/dh_t [T, B, H] (the head's derivative
    at each step, an input of the affine scan like the seed)."""
    T, B, _ = w.h.shape
    ys = _rng(seed + 7).integers(0, 10, size=(T, B))
    return np.stack([head_seed(w.h[t], w.params["W_out"], w.params["b_out"], ys[t]) for t in range(T)])


def norm_preserving_rnn(T: int, B: int, H: int, seed: int = 0):
    """W_hh = c Q (Q seeded orthogonal), h_t ~ U(-0.01, 0.01), c = 1/(1 - 0.01^2/3).

    Keeps |grad_h| O(|seed|) over the whole sequence (SURVEY 8(c) reading 12).
    """
    g = _rng(seed)
    Q, R = np.linalg.qr(g.standard_normal((H, H)))
    Q = Q * np.sign(np.diag(R))[None, :]
    c = 1.0 / (1.0 - 0.01 ** 2 / 3.0)
    W = (c * Q).astype(F32)
    h = g.uniform(-0.01, 0.01, size=(T, B, H)).astype(F32)
    seed_vec = g.standard_normal((B, H)).astype(F32)
    return dict(h=h, W_hh=W, g=seed_vec)


def int_rnn_family(T: int, B: int, H: int, seed: int = 0, p_sat: float = 0.002):
    """Integer family for the fused RNN leaf: W_hh a signed permutation and
    h_t in {0, +-1} so that 1-h^2 in {1, 0}; seed entries in [-8, 8].
    Every chain/tree value is an exact small integer in fp32."""
    g = _rng(seed)
    perm = g.permutation(H)
    sign = g.choice(np.array([-1.0, 1.0]), size=H)
    W = np.zeros((H, H), F32)
    W[np.arange(H), perm] = sign
    sat = g.random((T, B, H)) < p_sat
    h = np.where(sat, g.choice(np.array([-1.0, 1.0]), size=(T, B, H)), 0.0).astype(F32)
    s = g.integers(-8, 9, size=(B, H)).astype(F32)
    return dict(h=h, W_hh=W, g=s)


def int_dense_family(T: int, B: int, H: int, seed: int = 0, n_copy: int = 10,
                     p_merge: float = 0.02):
    """Integer transposed Jacobians J^T[t,b] (row-major), seed in [-4, 4].

    Each J^T is a signed 'column function' matrix (every column has at most one
    +-1), i.e. ||J^T||_1 <= 1, except for `n_copy` (t,b) positions overall where
    one column carries two +-1 entries (||.||_1 = 2).  'Merges' (two columns
    hitting one row) occur with probability p_merge per matrix.  Hence every
    product of any window of the chain has entries bounded by 2^n_copy and every
    partial sum of every GEMV is bounded by ||seed||_1 2^n_copy < 2^24: all
    associations are exact in fp32 (checked in tests/test_oracle_pins.py).
    """
    g = _rng(seed)
    JT = np.zeros((T, B, H, H), F32)
    copies = set()
    while len(copies) < min(n_copy, T * B):
        copies.add((int(g.integers(T)), int(g.integers(B))))
    for t in range(T):
        for b in range(B):
            tau = g.permutation(H)
            if g.random() < p_merge and H >= 2:
                k1, k2 = g.choice(H, size=2, replace=False)
                tau[k1] = tau[k2]          # two columns map to one row
            sgn = g.choice(np.array([-1.0, 1.0]), size=H)
            JT[t, b, tau, np.arange(H)] = sgn
            if (t, b) in copies and H >= 2:
                k = int(g.integers(H))
                other = (tau[k] + 1 + int(g.integers(H - 1))) % H
                JT[t, b, other, k] = g.choice(np.array([-1.0, 1.0]))
    s = g.integers(-4, 5, size=(B, H)).astype(F32)
    return dict(JT=JT, g=s)


def random_dense_family(T: int, B: int, H: int, seed: int = 0, gain: float = 1.0):
    """Dense random J^T with spectral scale ~gain (Gaussian / sqrt(H))."""
    g = _rng(seed)
    JT = (g.standard_normal((T, B, H, H)) * (gain / math.sqrt(H))).astype(F32)
    s = g.standard_normal((B, H)).astype(F32)
    return dict(JT=JT, g=s)


# --------------------------------------------------------------------------
# GRU, IRMAS-shaped data (Table 3)
# --------------------------------------------------------------------------

IRMAS_SETS = {"S": (259, 38), "M": (517, 24), "L": (1034, 12)}   # Table 3


def irmas_like(F: int, C: int, B: int, seed: int = 0, classes: int = 11):
    """x[f, b, :] ~ N(0.1 c_b, 1), then per-sample per-coefficient standardisation
    across frames (zero mean, unit variance)."""
    g = _rng(seed)
    labels = g.integers(0, classes, size=B)
    x = g.standard_normal((F, B, C)) + 0.1 * labels[None, :, None]
    x = (x - x.mean(axis=0, keepdims=True)) / x.std(axis=0, keepdims=True)
    return x.astype(F32), labels.astype(np.int64)


def gru_params(H: int, I: int, classes: int = 11, seed: int = 0):
    """torch nn.GRU layout: W_ih3 [3H, I], W_hh3 [3H, H] in (r, z, n) order."""
    g = _rng(seed)
    k = 1.0 / math.sqrt(H)
    u = lambda *s: g.uniform(-k, k, size=s).astype(F32)
    return dict(W_ih3=u(3 * H, I), W_hh3=u(3 * H, H), b_ih3=u(3 * H), b_hh3=u(3 * H),
                W_out=u(classes, H), b_out=u(classes))


def _sigmoid(v):
    return (1.0 / (1.0 + np.exp(-v))).astype(F32)


def gru_forward(x: np.ndarray, p: dict, h0: np.ndarray | None = None) -> dict:
    """fp32 forward of eqn:gru capturing the tape of P:826-831."""
    T, B, _ = x.shape
    H = p["W_hh3"].shape[1]
    h = np.zeros((B, H), F32) if h0 is None else h0.astype(F32).copy()
    gi = x @ p["W_ih3"].T + p["b_ih3"]                      # [T,B,3H]
    Whh_T = np.ascontiguousarray(p["W_hh3"].T)
    tape = {k: np.empty((T, B, H), F32) for k in ("h_prev", "r", "z", "n", "M", "h")}
    for t in range(T):
        gh = h @ Whh_T + p["b_hh3"]                           # [B,3H]
        r = _sigmoid(gi[t, :, :H] + gh[:, :H])
        z = _sigmoid(gi[t, :, H:2 * H] + gh[:, H:2 * H])
        M = gh[:, 2 * H:]
        n = np.tanh(gi[t, :, 2 * H:] + r * M).astype(F32)
        tape["h_prev"][t] = h
        h = ((1.0 - z) * n + z * h).astype(F32)
        tape["r"][t], tape["z"][t], tape["n"][t], tape["M"][t], tape["h"][t] = r, z, n, M, h
    return tape


@dataclass
class GruWorkload:
    x: np.ndarray
    labels: np.ndarray
    params: dict
    tape: dict
    g: np.ndarray


def gru_workload(set_name: str, B: int, H: int = 20, seed: int = 0) -> GruWorkload:
    F, C = IRMAS_SETS[set_name]
    x, labels = irmas_like(F, C, B, seed)
    p = gru_params(H, C, 11, seed + 1)
    tape = gru_forward(x, p)
    g = head_seed(tape["h"][-1], p["W_out"], p["b_out"], labels)
    return GruWorkload(x, labels, p, tape, g)


def gru_zero_family(T: int, B: int, H: int, seed: int = 0):
    """All weights/biases zero: r = z = 0.5, M = 0, n = 0 -> J^T = 0.5 I."""
    g = _rng(seed)
    zeros = np.zeros((T, B, H), F32)
    half = np.full((T, B, H), 0.5, F32)
    hp = g.integers(-4, 5, size=(T, B, H)).astype(F32)   # h_prev is irrelevant when W = 0
    tape = dict(h_prev=hp, r=half.copy(), z=half.copy(), n=zeros.copy(), M=zeros.copy())
    W = np.zeros((3 * H, H), F32)
    s = g.integers(-8, 9, size=(B, H)).astype(F32)
    return dict(tape=tape, W_hh3=W, g=s)


def gru_int_family(T: int, B: int, H: int, seed: int = 0, p_z: float = 0.03):
    """Gates chosen so every J^T is an exact signed column-function matrix:
    r = 1, n = 0, z in {0,1}: J^T[:, j] = z_j e_j + (1 - z_j) W_hn^T[:, j] with
    W_hn a signed permutation; W_hr, W_hz random integers (multiplied by exact
    zeros r(1-r) = z(1-z) = 0)."""
    g = _rng(seed)
    perm = g.permutation(H)
    W = np.zeros((3 * H, H), F32)
    W[:H] = g.integers(-3, 4, size=(H, H))
    W[H:2 * H] = g.integers(-3, 4, size=(H, H))
    W[2 * H + np.arange(H), perm] = g.choice(np.array([-1.0, 1.0]), size=H)
    z = (g.random((T, B, H)) < p_z).astype(F32)
    tape = dict(h_prev=g.integers(-4, 5, size=(T, B, H)).astype(F32),
                r=np.ones((T, B, H), F32), z=z,
                n=np.zeros((T, B, H), F32),
                M=g.integers(-4, 5, size=(T, B, H)).astype(F32))
    s = g.integers(-8, 9, size=(B, H)).astype(F32)
    return dict(tape=tape, W_hh3=W, g=s)


# --------------------------------------------------------------------------
# VGG-11 conv stack on 32x32x3 (config 5)
# --------------------------------------------------------------------------

VGG11_CFG = [64, "M", 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"]


def vgg11_ops(cfg=VGG11_CFG, in_ch: int = 3, hw: int = 32):
    """Operator list f_1..f_n of the conv part of VGG-11: ('conv', ci, co, h, w),
    ('relu', c, h, w), ('pool', c, h, w) with (h, w) the *input* spatial size."""
    ops, c, h = [], in_ch, hw
    for v in cfg:
        if v == "M":
            ops.append(("pool", c, h, h))
            h //= 2
        else:
            ops.append(("conv", c, v, h, h))
            ops.append(("relu", v, h, h))
            c = v
    return ops


def vgg11_pruned_weights(seed: int = 0, density: float = 0.03, cfg=VGG11_CFG):
    """Kaiming-normal 3x3 conv weights, per-layer magnitude pruning keeping the
    top `density` fraction (SURVEY reading 20: 97 % pruning, See et al. P:357)."""
    g = _rng(seed)
    ws, c = [], 3
    for v in cfg:
        if v == "M":
            continue
        std = math.sqrt(2.0 / (v * 9))
        w = (g.standard_normal((v, c, 3, 3)) * std).astype(F32)
        if density < 1.0:
            k = max(1, int(round(density * w.size)))
            thr = np.partition(np.abs(w).ravel(), w.size - k)[w.size - k]
            w = np.where(np.abs(w) >= thr, w, 0.0).astype(F32)
        ws.append(w)
        c = v
    return ws


def vgg11_forward(images: np.ndarray, weights, cfg=VGG11_CFG):
    """fp32 forward of the conv stack (torch CPU ops as plumbing).  Returns, per
    operator, the data the CSR Jacobian builders need: ReLU inputs (for the 0/1
    diagonal, Alg. 7) and flat pool indices within each channel plane (Alg. 8)."""
    import torch
    import torch.nn.functional as Fn
    x = torch.from_numpy(images)
    recs, wi = [], 0
    with torch.no_grad():
        for v in cfg:
            if v == "M":
                y, idx = Fn.max_pool2d(x, 2, 2, return_indices=True)
                recs.append(("pool", idx.numpy().astype(np.int64)))
                x = y
            else:
                x = Fn.conv2d(x, torch.from_numpy(weights[wi]), padding=1)
                recs.append(("conv", None))
                recs.append(("relu", x.numpy().copy()))
                x = torch.relu(x)
                wi += 1
    return recs, x.numpy()


def vgg11_workload(B: int = 16, seed: int = 0, density: float = 0.03):
    g = _rng(seed)
    images = g.standard_normal((B, 3, 32, 32)).astype(F32)
    weights = vgg11_pruned_weights(seed + 1, density)
    recs, out = vgg11_forward(images, weights)
    seed_vec = g.standard_normal((B, out[0].size)).astype(F32)
    return dict(images=images, weights=weights, recs=recs, ops=vgg11_ops(), g=seed_vec)
