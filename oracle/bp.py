"""Oracle: back-propagation by its plain definition, in fp64 (test infrastructure).

Notation: h_t = f_t(h_{t-1}) is the recurrent step, J_t = dh_t/dh_{t-1},
grad_h[t] = dl/dh_t (total derivative).  eqn:backprop:

    grad_h[t-1] = J_t^T grad_h[t],   t = T-1 ... 1,   grad_h[T-1] = seed

and dl/dh_init = J_0^T grad_h[0] is the optional inclusive extra (reading 3).
"""
from __future__ import annotations

import numpy as np

D = np.float64


def _d(a):
    return np.asarray(a, dtype=D)


# ---------------------------------------------------------------------------
# Leaf transposed Jacobians
# ---------------------------------------------------------------------------

def rnn_jt(h_t, W_hh):
    """J_t^T for eqn:rnn: h_t = tanh(... + W_hh h_{t-1}) gives
    J_t = diag(1 - h_t^2) W_hh, hence J_t^T = W_hh^T diag(1 - h_t^2)
    (reading 1).  h_t: [B,H] -> [B,H,H]."""
    h_t, W = _d(h_t), _d(W_hh)
    d = 1.0 - h_t * h_t
    return W.T[None, :, :] * d[:, None, :]          # scale column k by d_k


def gru_jt(h_prev, r, z, n, M, W_hh3):
    """J_t^T for the GRU, eqn:gru_jcb, read as the transpose with
    column broadcasting (reading 2):

      J^T = (W_hr^T o (j2 o j3)^T + W_hn^T o j5^T) o (j6 o j7)^T
            + W_hz^T o (j9 o j10)^T + J11
      j2 = r(1-r), j3 = M, j5 = r, j6 = 1-n^2, j7 = 1-z, j9 = z(1-z),
      j10 = h_{t-1} - n, J11 = I o z = diag(z)

    where "A o v^T" multiplies column j of A by v_j.  W_hh3 = [W_hr; W_hz; W_hn]
    (torch order r, z, n).  All gate arrays [B,H] -> [B,H,H]."""
    h_prev, r, z, n, M, W = map(_d, (h_prev, r, z, n, M, W_hh3))
    H = W.shape[1]
    W_hr, W_hz, W_hn = W[:H], W[H:2 * H], W[2 * H:]
    j2, j3, j5 = r * (1 - r), M, r
    j6, j7 = 1 - n * n, 1 - z
    j9, j10 = z * (1 - z), h_prev - n
    col = lambda A, v: A.T[None, :, :] * v[:, None, :]   # A^T o v^T
    inner = col(W_hr, j2 * j3) + col(W_hn, j5)
    JT = inner * (j6 * j7)[:, None, :] + col(W_hz, j9 * j10)
    idx = np.arange(H)
    JT[:, idx, idx] += z
    return JT


# ---------------------------------------------------------------------------
# Sequential BP (the plain definition; eqn:backprop P:86-88)
# ---------------------------------------------------------------------------

def bp_rnn(h, W_hh, seed):
    """grad_h[t] for all t and dl/dh_init for the tanh RNN.

    v <- seed; for t = T-1..0: grad_h[t] = v; v <- J_t^T v = W^T((1-h_t^2) o v).
    h: [T,B,H], W_hh: [H,H], seed: [B,H].  Returns (grad_h [T,B,H], grad_init [B,H]).
    """
    h, W, v = _d(h), _d(W_hh), _d(seed).copy()
    T = h.shape[0]
    out = np.empty(h.shape, D)
    for t in range(T - 1, -1, -1):
        out[t] = v
        v = ((1.0 - h[t] * h[t]) * v) @ W        # (J_t^T v)_i = sum_k W[k,i] d_k v_k
    return out, v


def bp_dense(JT, seed):
    """Sequential BP over explicit transposed Jacobians JT[t] = J_t^T ([T,B,H,H])."""
    JT, v = _d(JT), _d(seed).copy()
    T = JT.shape[0]
    out = np.empty((T,) + v.shape, D)
    for t in range(T - 1, -1, -1):
        out[t] = v
        v = np.einsum("bik,bk->bi", JT[t], v)
    return out, v


def bp_gru(tape, W_hh3, seed):
    """Sequential BP for the GRU using eqn:gru_jcb leaves."""
    v = _d(seed).copy()
    T = tape["r"].shape[0]
    out = np.empty((T,) + v.shape, D)
    for t in range(T - 1, -1, -1):
        out[t] = v
        JT = gru_jt(tape["h_prev"][t], tape["r"][t], tape["z"][t], tape["n"][t],
                    tape["M"][t], W_hh3)
        v = np.einsum("bik,bk->bi", JT, v)
    return out, v


# ---------------------------------------------------------------------------
# Per-step losses: the affine recurrence (reading 8 notes
# the paper covers the last-step loss only).  With l = sum_t l_t(h_t)
# and e_t = dl_t/dh_t (partial), the total derivative obeys
#     grad_h[T-1] = seed + e_{T-1},   grad_h[t-1] = J_t^T grad_h[t] + e_{t-1},
# and dl/dh_init = J_0^T grad_h[0] (no e_{-1}).  As a scan: elements (J^T, e)
# composed by (A, a) <> (B, b) = (BA, Ba + b).
# ---------------------------------------------------------------------------

def bp_affine(jt, T, seed, e):
    """Sequential affine BP; jt(t) -> J_t^T [B,H,H]; e: [T,B,H]."""
    e = _d(e)
    v = _d(seed) + e[T - 1]
    out = np.empty((T,) + v.shape, D)
    for t in range(T - 1, -1, -1):
        out[t] = v
        v = np.einsum("bik,bk->bi", jt(t), v)
        if t >= 1:
            v = v + e[t - 1]
    return out, v


def bp_rnn_affine(h, W_hh, seed, e):
    return bp_affine(lambda t: rnn_jt(h[t], W_hh), len(h), seed, e)


def bp_dense_affine(JT, seed, e):
    return bp_affine(lambda t: _d(JT[t]), len(JT), seed, e)


def bp_gru_affine(tape, W_hh3, seed, e):
    return bp_affine(lambda t: gru_jt(tape["h_prev"][t], tape["r"][t], tape["z"][t], tape["n"][t],
                                      tape["M"][t], W_hh3), len(tape["r"]), seed, e)


# ---------------------------------------------------------------------------
# Parameter gradients, eqn:update_param with tied weights summed over
# time: each time step is a layer sharing theta.
# ---------------------------------------------------------------------------

def weight_grads_rnn(x, h, grad_h, h_init=None):
    """delta_t = (1 - h_t^2) o grad_h[t];  dW_hh = sum_{t,b} delta_t h_{t-1}^T,
    dW_ih = sum delta_t x_t^T, db_ih = db_hh = sum delta_t (reading 9)."""
    x, h, gh = _d(x), _d(h), _d(grad_h)
    T, B, H = h.shape
    hp = np.zeros((T, B, H), D)
    hp[1:] = h[:-1]
    if h_init is not None:
        hp[0] = _d(h_init)
    delta = (1.0 - h * h) * gh
    dW_hh = np.einsum("tbi,tbk->ik", delta, hp)
    dW_ih = np.einsum("tbi,tbj->ij", delta, x)
    db = delta.sum(axis=(0, 1))
    return dW_ih, dW_hh, db


def weight_grads_gru(x, tape, grad_h):
    """Per-gate deltas of the eqn:gru_rewrite form:
      dN = g o (1-z) o (1-n^2)            (through n = tanh N)
      dZ = g o (h_{t-1}-n) o z(1-z)       (through z = sigma Z)
      dR = dN o M o r(1-r)                (through r = sigma R, N = ... + r o M)
      dM = dN o r                         (M = W_hn h_{t-1} + b_hn)
    dW_ih3 = [dR; dZ; dN] x^T, dW_hh3 = [dR; dZ; dM] h_{t-1}^T,
    db_ih3 = sum [dR; dZ; dN], db_hh3 = sum [dR; dZ; dM]."""
    x, g = _d(x), _d(grad_h)
    hp, r, z, n, M = (_d(tape[k]) for k in ("h_prev", "r", "z", "n", "M"))
    dN = g * (1 - z) * (1 - n * n)
    dZ = g * (hp - n) * z * (1 - z)
    dR = dN * M * r * (1 - r)
    dM = dN * r
    gi = np.concatenate([dR, dZ, dN], axis=2)
    gh = np.concatenate([dR, dZ, dM], axis=2)
    dW_ih3 = np.einsum("tbi,tbj->ij", gi, x)
    dW_hh3 = np.einsum("tbi,tbj->ij", gh, hp)
    return dW_ih3, dW_hh3, gi.sum(axis=(0, 1)), gh.sum(axis=(0, 1))


# ---------------------------------------------------------------------------
# fp64 forward + loss (used only by the finite-difference pins)
# ---------------------------------------------------------------------------

def rnn_forward64(x, p, h0=None, t_start=0, h_start=None):
    """eqn:rnn in fp64.  If h_start is given, the recurrence restarts at step
    t_start+1 from h_{t_start} = h_start (used to perturb a hidden state)."""
    x = _d(x)
    T, B, _ = x.shape
    Wih, Whh = _d(p["W_ih"]), _d(p["W_hh"])
    b = _d(p["b_ih"]) + _d(p["b_hh"])
    H = Whh.shape[0]
    hs = np.empty((T, B, H), D)
    if h_start is None:
        h = np.zeros((B, H), D) if h0 is None else _d(h0).copy()
        t0 = 0
    else:
        h = _d(h_start).copy()
        hs[t_start] = h
        t0 = t_start + 1
    for t in range(t0, T):
        h = np.tanh(x[t] @ Wih.T + b + h @ Whh.T)
        hs[t] = h
    return hs


def ce_loss64(h_last, W_out, b_out, labels):
    """Mean softmax cross-entropy over the batch (reading 6)."""
    logits = _d(h_last) @ _d(W_out).T + _d(b_out)
    m = logits.max(axis=1, keepdims=True)
    lse = (m[:, 0] + np.log(np.exp(logits - m).sum(axis=1)))
    return float(np.mean(lse - logits[np.arange(len(labels)), labels]))


def seed64(h_last, W_out, b_out, labels):
    """dl/dh_{T-1} of ce_loss64 (closed form softmax - onehot, /B)."""
    logits = _d(h_last) @ _d(W_out).T + _d(b_out)
    logits -= logits.max(axis=1, keepdims=True)
    pr = np.exp(logits)
    pr /= pr.sum(axis=1, keepdims=True)
    pr[np.arange(len(labels)), labels] -= 1.0
    return pr @ _d(W_out) / len(labels)


def gru_forward64(x, p, h0=None, t_start=0, h_start=None):
    """eqn:gru in fp64, returning the tape of P:826-831."""
    x = _d(x)
    T, B, _ = x.shape
    Wih, Whh = _d(p["W_ih3"]), _d(p["W_hh3"])
    bih, bhh = _d(p["b_ih3"]), _d(p["b_hh3"])
    H = Whh.shape[1]
    sig = lambda v: 1.0 / (1.0 + np.exp(-v))
    tape = {k: np.zeros((T, B, H), D) for k in ("h_prev", "r", "z", "n", "M", "h")}
    if h_start is None:
        h = np.zeros((B, H), D) if h0 is None else _d(h0).copy()
        t0 = 0
    else:
        h = _d(h_start).copy()
        tape["h"][t_start] = h
        t0 = t_start + 1
    for t in range(t0, T):
        gi = x[t] @ Wih.T + bih
        gh = h @ Whh.T + bhh
        r = sig(gi[:, :H] + gh[:, :H])
        z = sig(gi[:, H:2 * H] + gh[:, H:2 * H])
        M = gh[:, 2 * H:]
        n = np.tanh(gi[:, 2 * H:] + r * M)
        tape["h_prev"][t] = h
        h = (1 - z) * n + z * h
        tape["r"][t], tape["z"][t], tape["n"][t], tape["M"][t], tape["h"][t] = r, z, n, M, h
    return tape


def gru_gates64(x, h, p, h_init=None):
    """The GRU 'forward overhead' (FO; reading 10): the tape of
    P:826-831 recomputed from given h_0..h_{T-1} — eqn:gru's gate formulas at
    h_prev[t] = h[t-1] (h_init, default 0, at t = 0), no recurrence."""
    x, h = _d(x), _d(h)
    T, B, _ = x.shape
    Wih, Whh = _d(p["W_ih3"]), _d(p["W_hh3"])
    bih, bhh = _d(p["b_ih3"]), _d(p["b_hh3"])
    H = Whh.shape[1]
    hp = np.concatenate([(np.zeros((1, B, H), D) if h_init is None else _d(h_init)[None]), h[:-1]], axis=0)
    gi = x @ Wih.T + bih
    gh = hp @ Whh.T + bhh
    sig = lambda v: 1.0 / (1.0 + np.exp(-v))
    r = sig(gi[..., :H] + gh[..., :H])
    z = sig(gi[..., H:2 * H] + gh[..., H:2 * H])
    M = gh[..., 2 * H:]
    n = np.tanh(gi[..., 2 * H:] + r * M)
    return {"h_prev": hp, "r": r, "z": z, "n": n, "M": M}

