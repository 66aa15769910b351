"""Pins for the oracle's affine recurrence (per-step losses, SURVEY 8(f)
NEXT-4; not in the paper, whose loss sits on the last step only):
torch.autograd fp64 with a loss on every step (retain_grad on every h_t),
closed forms, and reduction to the plain BP of eqn:backprop."""
import math

import numpy as np
import torch

import bppsa_workloads as W
from oracle import bp

RNG = np.random.default_rng(99)


def test_rnn_affine_vs_torch_autograd():
    """Loss = sum_t CE(W_out h_t + b_out, y_t): e_t is the per-step head
    gradient (seed64 at each t); the oracle's affine BP equals autograd's
    total derivatives dl/dh_t and dl/dh_init."""
    T, H, I, B = 25, 20, 1, 3
    w = W.rnn_workload(T, B, H, seed=8)
    cell = torch.nn.RNNCell(I, H, nonlinearity="tanh").double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(w.params["W_ih"]))
        cell.weight_hh.copy_(torch.from_numpy(w.params["W_hh"]))
        cell.bias_ih.copy_(torch.from_numpy(w.params["b_ih"]))
        cell.bias_hh.copy_(torch.from_numpy(w.params["b_hh"]))
    Wo, bo = w.params["W_out"], w.params["b_out"]
    ys = RNG.integers(0, 10, (T, B))
    x = torch.from_numpy(w.x.astype(np.float64))
    h0 = torch.zeros(B, H, dtype=torch.float64, requires_grad=True)
    hs, hcur = [], h0
    for t in range(T):
        hcur = cell(x[t], hcur)
        hcur.retain_grad()
        hs.append(hcur)
    loss = sum(torch.nn.functional.cross_entropy(hs[t] @ torch.from_numpy(Wo).double().T
                                                 + torch.from_numpy(bo).double(), torch.from_numpy(ys[t]))
               for t in range(T))
    loss.backward()
    h64 = torch.stack([v.detach() for v in hs]).numpy()
    e = np.stack([bp.seed64(h64[t], Wo, bo, ys[t]) for t in range(T)])
    grad, gi = bp.bp_rnn_affine(h64, w.params["W_hh"], np.zeros((B, H)), e)
    assert np.abs(grad - torch.stack([v.grad for v in hs]).numpy()).max() < 1e-12
    assert np.abs(gi - h0.grad.numpy()).max() < 1e-12


def test_gru_affine_vs_torch_autograd():
    T, B, H, C = 15, 2, 20, 12
    k = 1 / math.sqrt(H)
    u = lambda *s: RNG.uniform(-k, k, size=s) * 2
    p = dict(W_ih3=u(3 * H, C), W_hh3=u(3 * H, H), b_ih3=u(3 * H), b_hh3=u(3 * H))
    x = RNG.standard_normal((T, B, C))
    c = RNG.standard_normal((T, B, H))                     # loss = sum_t <c_t, h_t>  =>  e_t = c_t
    cell = torch.nn.GRUCell(C, H).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(p["W_ih3"]))
        cell.weight_hh.copy_(torch.from_numpy(p["W_hh3"]))
        cell.bias_ih.copy_(torch.from_numpy(p["b_ih3"]))
        cell.bias_hh.copy_(torch.from_numpy(p["b_hh3"]))
    hs, hcur = [], torch.zeros(B, H, dtype=torch.float64)
    for t in range(T):
        hcur = cell(torch.from_numpy(x[t]), hcur)
        hcur.retain_grad()
        hs.append(hcur)
    sum((hs[t] * torch.from_numpy(c[t])).sum() for t in range(T)).backward()
    tape = bp.gru_forward64(x, p)
    grad, _ = bp.bp_gru_affine(tape, p["W_hh3"], np.zeros((B, H)), c)
    assert np.abs(grad - torch.stack([v.grad for v in hs]).numpy()).max() < 1e-12


def test_affine_closed_forms_and_reductions():
    T, B, H = 40, 2, 7
    h = RNG.uniform(-0.9, 0.9, (T, B, H))
    Wm = RNG.standard_normal((H, H)) * 0.4
    g = RNG.standard_normal((B, H))
    e = RNG.standard_normal((T, B, H))
    # e = 0: plain BP (eqn:backprop)
    a, ai = bp.bp_rnn_affine(h, Wm, g, np.zeros_like(e))
    r, ri = bp.bp_rnn(h, Wm, g)
    assert np.abs(a - r).max() <= 1e-13 * np.abs(r).max() and np.abs(ai - ri).max() <= 1e-13 * np.abs(r).max()
    # W_hh = 0: only the step's own loss survives
    z, zi = bp.bp_rnn_affine(h, np.zeros((H, H)), g, e)
    assert np.array_equal(z[:-1], e[:-1]) and np.allclose(z[-1], g + e[-1], rtol=0, atol=0)
    assert not zi.any()
    # linearity in (seed, e)
    s1, _ = bp.bp_rnn_affine(h, Wm, g, np.zeros_like(e))
    s2, _ = bp.bp_rnn_affine(h, Wm, np.zeros_like(g), e)
    s, _ = bp.bp_rnn_affine(h, Wm, g, e)
    assert np.abs(s - (s1 + s2)).max() < 1e-12
    # dense leaves == fused RNN leaves
    JT = np.stack([bp.rnn_jt(h[t], Wm) for t in range(T)])
    d, di = bp.bp_dense_affine(JT, g, e)
    assert np.abs(d - s).max() < 1e-12
