"""Pins for oracle/bp.py against things other than itself: finite differences,
brute-force explicit products, closed forms, torch.autograd (fp64, CPU)."""
import math

import numpy as np
import pytest
import torch

import bppsa_workloads as W
from oracle import bp

RNG = np.random.default_rng(1234)


def _rnn_params64(H, I, C, rng):
    k = 1 / math.sqrt(H)
    u = lambda *s: rng.uniform(-k, k, size=s)
    return dict(W_ih=u(H, I), W_hh=u(H, H) * 3, b_ih=u(H), b_hh=u(H), W_out=u(C, H), b_out=u(C))


def _gru_params64(H, I, C, rng):
    k = 1 / math.sqrt(H)
    u = lambda *s: rng.uniform(-k, k, size=s) * 2
    return dict(W_ih3=u(3 * H, I), W_hh3=u(3 * H, H), b_ih3=u(3 * H), b_hh3=u(3 * H),
                W_out=u(C, H), b_out=u(C))


# ---------------------------------------------------------------- leaf J^T

def test_rnn_jt_vs_finite_differences():
    """J_t^T = W^T diag(1-h^2) vs central differences of one RNN step."""
    H, I, B = 20, 3, 2
    p = _rnn_params64(H, I, 10, RNG)
    hprev = RNG.uniform(-1, 1, (B, H))
    x = RNG.standard_normal((B, I))
    step = lambda hp: np.tanh(x @ p["W_ih"].T + p["b_ih"] + p["b_hh"] + hp @ p["W_hh"].T)
    h = step(hprev)
    JT = bp.rnn_jt(h, p["W_hh"])
    eps = 1e-6
    for b in range(B):
        J_fd = np.zeros((H, H))
        for k in range(H):
            e = np.zeros((B, H)); e[b, k] = eps
            J_fd[:, k] = (step(hprev + e)[b] - step(hprev - e)[b]) / (2 * eps)   # J[i,k] = dh_i/dhp_k
        assert np.abs(JT[b] - J_fd.T).max() < 1e-5
        # the north_star's literal "diag(1-h^2) W_hh" is J, not J^T (reading 1)
        assert np.abs(JT[b] - J_fd).max() > 1e-3


def test_rnn_jt_special_cases():
    H = 7
    Wm = RNG.standard_normal((H, H))
    assert np.array_equal(bp.rnn_jt(np.zeros((1, H)), Wm)[0], Wm.T)       # h = 0 -> W^T
    assert not bp.rnn_jt(RNG.uniform(-1, 1, (2, H)), np.zeros((H, H))).any()  # W = 0 -> 0


@pytest.mark.parametrize("case", range(100))
def test_gru_jt_vs_finite_differences(case):
    """eqn:gru_jcb, transposed reading (reading 2), vs central differences of the
    full GRU cell (eqn:gru) within 1e-5 over 100 random cases."""
    rng = np.random.default_rng(case)
    H, I, B = (20, 4, 1) if case < 90 else (int(rng.integers(1, 9)), 3, 2)
    p = _gru_params64(H, I, 11, rng)
    x = rng.standard_normal((1, B, I))
    hprev = rng.uniform(-1, 1, (B, H))
    tape = bp.gru_forward64(x, p, h0=hprev)
    JT = bp.gru_jt(hprev, tape["r"][0], tape["z"][0], tape["n"][0], tape["M"][0], p["W_hh3"])
    eps = 1e-6
    for b in range(B):
        J = np.zeros((H, H))
        for k in range(H):
            e = np.zeros((B, H)); e[b, k] = eps
            hp = bp.gru_forward64(x, p, h0=hprev + e)["h"][0, b]
            hm = bp.gru_forward64(x, p, h0=hprev - e)["h"][0, b]
            J[:, k] = (hp - hm) / (2 * eps)
        assert np.abs(JT[b] - J.T).max() < 1e-5
        if H > 1:
            assert np.abs(JT[b] - J).max() > 1e-4 or np.abs(J - J.T).max() < 1e-4


def test_gru_jt_zero_weights_is_half_identity():
    """all-zero weights -> r = z = 0.5, M = n = 0 -> J^T = 0.5 I exactly."""
    H, B = 20, 3
    p = {k: np.zeros_like(v) for k, v in _gru_params64(H, 5, 11, RNG).items()}
    x = RNG.standard_normal((1, B, 5))
    hprev = RNG.standard_normal((B, H))
    tape = bp.gru_forward64(x, p, h0=hprev)
    JT = bp.gru_jt(hprev, tape["r"][0], tape["z"][0], tape["n"][0], tape["M"][0], p["W_hh3"])
    assert np.array_equal(JT, np.broadcast_to(0.5 * np.eye(H), JT.shape))


# ---------------------------------------------------------------- sequential BP

def _rnn_case(T, H, I, B, rng):
    p = _rnn_params64(H, I, 10, rng)
    x = rng.standard_normal((T, B, I))
    labels = rng.integers(0, 10, B)
    h = bp.rnn_forward64(x, p)
    return p, x, labels, h


def test_bp_rnn_vs_finite_differences():
    """grad_h[t] = dl/dh_t (total derivative) vs central differences of the loss
    with h_t perturbed and the recurrence re-run from t+1 (T=10, H=20; <= 1e-6)."""
    T, H, I, B = 10, 20, 1, 2
    p, x, labels, h = _rnn_case(T, H, I, B, RNG)
    g = bp.seed64(h[-1], p["W_out"], p["b_out"], labels)
    grad, grad_init = bp.bp_rnn(h, p["W_hh"], g)
    eps = 1e-6
    loss_from = lambda t, ht: bp.ce_loss64(
        bp.rnn_forward64(x, p, t_start=t, h_start=ht)[-1], p["W_out"], p["b_out"], labels)
    worst = 0.0
    for t in range(T):
        for b in range(B):
            for i in range(H):
                e = np.zeros((B, H)); e[b, i] = eps
                fd = (loss_from(t, h[t] + e) - loss_from(t, h[t] - e)) / (2 * eps)
                worst = max(worst, abs(fd - grad[t, b, i]))
    assert worst < 1e-6
    # dl/dh_init
    for b in range(B):
        for i in range(H):
            e = np.zeros((B, H)); e[b, i] = eps
            lp = bp.ce_loss64(bp.rnn_forward64(x, p, h0=e)[-1], p["W_out"], p["b_out"], labels)
            lm = bp.ce_loss64(bp.rnn_forward64(x, p, h0=-e)[-1], p["W_out"], p["b_out"], labels)
            assert abs((lp - lm) / (2 * eps) - grad_init[b, i]) < 1e-6


def test_seed_vs_finite_differences():
    H, B = 20, 3
    p = _rnn_params64(H, 1, 10, RNG)
    hl = RNG.uniform(-1, 1, (B, H))
    labels = RNG.integers(0, 10, B)
    g = bp.seed64(hl, p["W_out"], p["b_out"], labels)
    eps = 1e-6
    for b in range(B):
        for i in range(H):
            e = np.zeros((B, H)); e[b, i] = eps
            fd = (bp.ce_loss64(hl + e, p["W_out"], p["b_out"], labels)
                  - bp.ce_loss64(hl - e, p["W_out"], p["b_out"], labels)) / (2 * eps)
            assert abs(fd - g[b, i]) < 1e-8
    # the generator's fp32 head_seed is the same quantity (input side)
    g32 = W.head_seed(hl.astype(np.float32), p["W_out"].astype(np.float32),
                      p["b_out"].astype(np.float32), labels)
    assert np.abs(g32 - g).max() < 1e-6


def test_bp_brute_force_explicit_products():
    """P2: P_t = J_{t+1}^T ... J_{T-1}^T as explicit fp64 matrices, P_t g == chain."""
    T, H, B = 12, 6, 2
    h = RNG.uniform(-1, 1, (T, B, H))
    Wm = RNG.standard_normal((H, H))
    g = RNG.standard_normal((B, H))
    grad, _ = bp.bp_rnn(h, Wm, g)
    JT = np.stack([bp.rnn_jt(h[t], Wm) for t in range(T)])
    for t in range(T):
        for b in range(B):
            P = np.eye(H)
            for s in range(t + 1, T):
                P = P @ JT[s, b]
            assert np.abs(P @ g[b] - grad[t, b]).max() < 1e-12 * max(1, np.abs(grad[t, b]).max())
    gd, _ = bp.bp_dense(JT, g)
    assert np.allclose(gd, grad, rtol=1e-13, atol=0)


def test_bp_closed_forms():
    """P4: W = 0 -> grad_h[t < T-1] = 0;  h = 0 -> grad_h[t] = (W^T)^{T-1-t} g."""
    T, H, B = 9, 5, 2
    g = RNG.standard_normal((B, H))
    grad, _ = bp.bp_rnn(RNG.uniform(-1, 1, (T, B, H)), np.zeros((H, H)), g)
    assert np.array_equal(grad[-1], g) and not grad[:-1].any()
    Wm = RNG.integers(-2, 3, (H, H)).astype(float)
    grad, _ = bp.bp_rnn(np.zeros((T, B, H)), Wm, g)
    for t in range(T):
        ref = g @ np.linalg.matrix_power(Wm, T - 1 - t)       # ((W^T)^k g)^T = g^T W^k
        assert np.allclose(grad[t], ref, rtol=1e-12, atol=1e-12)


def test_all_zero_rnn_loss_is_ln10():
    """all-zero parameters -> h = 0, uniform softmax over 10 classes."""
    T, H, B = 5, 20, 4
    p = {k: np.zeros_like(v) for k, v in _rnn_params64(H, 1, 10, RNG).items()}
    x = RNG.integers(0, 2, (T, B, 1)).astype(float)
    h = bp.rnn_forward64(x, p)
    assert not h.any()
    assert abs(bp.ce_loss64(h[-1], p["W_out"], p["b_out"], RNG.integers(0, 10, B)) - math.log(10)) < 1e-15


# ---------------------------------------------------------------- weight grads

def test_weight_grads_rnn_vs_finite_differences():
    T, H, I, B = 8, 6, 2, 2
    p, x, labels, h = _rnn_case(T, H, I, B, RNG)
    g = bp.seed64(h[-1], p["W_out"], p["b_out"], labels)
    grad, _ = bp.bp_rnn(h, p["W_hh"], g)
    dWih, dWhh, db = bp.weight_grads_rnn(x, h, grad)
    eps = 1e-6

    def L(q):
        return bp.ce_loss64(bp.rnn_forward64(x, q)[-1], q["W_out"], q["b_out"], labels)

    for name, ref in (("W_ih", dWih), ("W_hh", dWhh), ("b_ih", db), ("b_hh", db)):
        it = np.nditer(p[name], flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            qp = {k: v.copy() for k, v in p.items()}
            qm = {k: v.copy() for k, v in p.items()}
            qp[name][idx] += eps
            qm[name][idx] -= eps
            assert abs((L(qp) - L(qm)) / (2 * eps) - ref[idx]) < 1e-6, (name, idx)


def test_weight_grads_gru_vs_finite_differences():
    T, H, I, B = 6, 4, 3, 2
    p = _gru_params64(H, I, 11, RNG)
    x = RNG.standard_normal((T, B, I))
    labels = RNG.integers(0, 11, B)
    tape = bp.gru_forward64(x, p)
    g = bp.seed64(tape["h"][-1], p["W_out"], p["b_out"], labels)
    grad, _ = bp.bp_gru(tape, p["W_hh3"], g)
    dWih, dWhh, dbih, dbhh = bp.weight_grads_gru(x, tape, grad)
    eps = 1e-6

    def L(q):
        return bp.ce_loss64(bp.gru_forward64(x, q)["h"][-1], q["W_out"], q["b_out"], labels)

    for name, ref in (("W_ih3", dWih), ("W_hh3", dWhh), ("b_ih3", dbih), ("b_hh3", dbhh)):
        it = np.nditer(p[name], flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            qp = {k: v.copy() for k, v in p.items()}
            qm = {k: v.copy() for k, v in p.items()}
            qp[name][idx] += eps
            qm[name][idx] -= eps
            assert abs((L(qp) - L(qm)) / (2 * eps) - ref[idx]) < 1e-6, (name, idx)


def test_bp_gru_vs_finite_differences():
    T, H, I, B = 7, 5, 3, 2
    p = _gru_params64(H, I, 11, RNG)
    x = RNG.standard_normal((T, B, I))
    labels = RNG.integers(0, 11, B)
    tape = bp.gru_forward64(x, p)
    g = bp.seed64(tape["h"][-1], p["W_out"], p["b_out"], labels)
    grad, _ = bp.bp_gru(tape, p["W_hh3"], g)
    eps = 1e-6
    for t in range(T):
        for b in range(B):
            for i in range(H):
                e = np.zeros((B, H)); e[b, i] = eps
                lp = bp.ce_loss64(bp.gru_forward64(x, p, t_start=t, h_start=tape["h"][t] + e)["h"][-1],
                                  p["W_out"], p["b_out"], labels)
                lm = bp.ce_loss64(bp.gru_forward64(x, p, t_start=t, h_start=tape["h"][t] - e)["h"][-1],
                                  p["W_out"], p["b_out"], labels)
                assert abs((lp - lm) / (2 * eps) - grad[t, b, i]) < 1e-6


# ---------------------------------------------------------------- torch.autograd (P6)

def test_rnn_vs_torch_autograd():
    """P6: torch.autograd fp64 with an explicit RNNCell loop and retain_grad on
    every h_t (the paper's own baseline) gives the same grad_h and weight
    gradients."""
    T, H, I, B = 30, 20, 1, 4
    w = W.rnn_workload(T, B, H, seed=3)
    cell = torch.nn.RNNCell(I, H, nonlinearity="tanh").double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(w.params["W_ih"]))
        cell.weight_hh.copy_(torch.from_numpy(w.params["W_hh"]))
        cell.bias_ih.copy_(torch.from_numpy(w.params["b_ih"]))
        cell.bias_hh.copy_(torch.from_numpy(w.params["b_hh"]))
    x = torch.from_numpy(w.x.astype(np.float64))
    hs, hcur = [], torch.zeros(B, H, dtype=torch.float64)
    for t in range(T):
        hcur = cell(x[t], hcur)
        hcur.retain_grad()
        hs.append(hcur)
    logits = hs[-1] @ torch.from_numpy(w.params["W_out"]).double().T + torch.from_numpy(w.params["b_out"]).double()
    loss = torch.nn.functional.cross_entropy(logits, torch.from_numpy(w.labels))
    loss.backward()
    h64 = torch.stack([v.detach() for v in hs]).numpy()
    g = bp.seed64(h64[-1], w.params["W_out"], w.params["b_out"], w.labels)
    grad, _ = bp.bp_rnn(h64, w.params["W_hh"], g)
    ref = torch.stack([v.grad for v in hs]).numpy()
    assert np.abs(grad - ref).max() < 1e-12
    dWih, dWhh, db = bp.weight_grads_rnn(w.x, h64, grad)
    assert np.abs(dWhh - cell.weight_hh.grad.numpy()).max() < 1e-12
    assert np.abs(dWih - cell.weight_ih.grad.numpy()).max() < 1e-12
    assert np.abs(db - cell.bias_hh.grad.numpy()).max() < 1e-12


def test_gru_vs_torch_autograd():
    T, B = 25, 3
    H, C = 20, 12
    x = RNG.standard_normal((T, B, C))
    p = _gru_params64(H, C, 11, RNG)
    labels = RNG.integers(0, 11, B)
    cell = torch.nn.GRUCell(C, H).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(p["W_ih3"]))
        cell.weight_hh.copy_(torch.from_numpy(p["W_hh3"]))
        cell.bias_ih.copy_(torch.from_numpy(p["b_ih3"]))
        cell.bias_hh.copy_(torch.from_numpy(p["b_hh3"]))
    xt = torch.from_numpy(x)
    hs, hcur = [], torch.zeros(B, H, dtype=torch.float64)
    for t in range(T):
        hcur = cell(xt[t], hcur)
        hcur.retain_grad()
        hs.append(hcur)
    logits = hs[-1] @ torch.from_numpy(p["W_out"]).T + torch.from_numpy(p["b_out"])
    torch.nn.functional.cross_entropy(logits, torch.from_numpy(labels)).backward()
    tape = bp.gru_forward64(x, p)
    assert np.abs(tape["h"] - torch.stack([v.detach() for v in hs]).numpy()).max() < 1e-12
    g = bp.seed64(tape["h"][-1], p["W_out"], p["b_out"], labels)
    grad, _ = bp.bp_gru(tape, p["W_hh3"], g)
    assert np.abs(grad - torch.stack([v.grad for v in hs]).numpy()).max() < 1e-12
    dWih, dWhh, dbih, dbhh = bp.weight_grads_gru(x, tape, grad)
    assert np.abs(dWhh - cell.weight_hh.grad.numpy()).max() < 1e-12
    assert np.abs(dWih - cell.weight_ih.grad.numpy()).max() < 1e-12
    assert np.abs(dbih - cell.bias_ih.grad.numpy()).max() < 1e-12
    assert np.abs(dbhh - cell.bias_hh.grad.numpy()).max() < 1e-12


def test_generator_forward_matches_fp64_forward():
    """The fp32 input generator runs eqn:rnn / eqn:gru (inputs side); sanity-check
    against the oracle's fp64 forward."""
    w = W.rnn_workload(50, 3, 20, seed=5)
    h64 = bp.rnn_forward64(w.x, w.params)
    assert np.abs(h64 - w.h).max() < 1e-5
    gw = W.gru_workload("S", 2, seed=6)
    t64 = bp.gru_forward64(gw.x, gw.params)
    for k in ("h_prev", "r", "z", "n", "M", "h"):
        assert np.abs(t64[k] - gw.tape[k]).max() < 1e-4


def test_gru_gates_recompute_equals_the_forward_tape():
    """FO (reading 10): the gates recomputed from the forward's own h equal the
    tape the sequential fp64 forward recorded (gru_forward64, itself pinned by
    torch.autograd above), with and without h_init."""
    T, B, H, C = 30, 3, 20, 12
    p = _gru_params64(H, C, 11, RNG)
    x = RNG.standard_normal((T, B, C))
    for h0 in (None, RNG.standard_normal((B, H)) * 0.3):
        tape = bp.gru_forward64(x, p, h0=h0)
        g = bp.gru_gates64(x, tape["h"], p, h_init=h0)
        for k in ("h_prev", "r", "z", "n", "M"):
            assert np.abs(g[k] - tape[k]).max() < 1e-14, k
