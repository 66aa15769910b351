"""End-to-end training with the BPPSA backward: the same
model, data and optimizer as torch autograd (cuDNN backward), only the
backward differs, so the trajectories agree up to fp32 association."""
import copy

import numpy as np
import pytest
import torch

import bppsa_workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,B,H", [(2000, 16, 20), (1500, 16, 64), (777, 5, 32)])
def test_bppsa_training_matches_autograd(lib, T, B, H):
    from paper_1907_10134_b200.train import AutogradTrainer, BitstreamRnn, BppsaTrainer
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.manual_seed(0)
    ma = BitstreamRnn(H=H).cuda()
    mb = copy.deepcopy(ma)
    mb.rnn.flatten_parameters()
    ta, tb = BppsaTrainer(ma, lr=1e-3, block0=64), AutogradTrainer(mb, lr=1e-3)
    la, lb = [], []
    for it in range(25):
        x, y = W.bitstreams(T, B, seed=100 + it)
        x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        la.append(ta.step(x, y))
        lb.append(tb.step(x, y))
        if it == 0:     # identical forward and head; the BPPSA gradients == autograd's
            assert la[0] == pytest.approx(lb[0], rel=1e-6)
    la, lb = np.array(la), np.array(lb)
    assert np.abs(la - lb).max() <= 1e-3 * np.abs(lb).max(), (la, lb)
    for pa, pb in zip(ma.parameters(), mb.parameters()):
        d = (pa - pb).abs().max().item()
        assert d <= 1e-3 * max(pb.abs().max().item(), 1e-3), d


def test_bppsa_gradients_equal_autograd(lib):
    """One backward, no update: every parameter gradient within 1e-4 (max-norm
    relative) of torch autograd's."""
    from paper_1907_10134_b200 import api
    torch.backends.cudnn.allow_tf32 = False
    T, B, H = 3000, 8, 64
    torch.manual_seed(3)
    from paper_1907_10134_b200.train import BitstreamRnn
    m = BitstreamRnn(H=H).cuda()
    x, y = W.bitstreams(T, B, seed=5)
    x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    h, logits = m(x)
    torch.nn.functional.cross_entropy(logits, y).backward()
    ref = {n: p.grad.clone() for n, p in m.rnn.named_parameters()}
    with torch.no_grad():
        h, _ = m.rnn(x)
    hl = h[-1].detach().requires_grad_(True)
    torch.nn.functional.cross_entropy(m.head(hl), y).backward()
    jac = api.jacobians_rnn(h.contiguous(), m.rnn.weight_hh_l0.detach().contiguous())
    grad, _ = api.scan(jac, hl.grad.contiguous())
    dWih, dWhh, db = api.weight_grads_rnn(x, h.contiguous(), grad)
    got = {"weight_ih_l0": dWih, "weight_hh_l0": dWhh, "bias_ih_l0": db, "bias_hh_l0": db}
    for n, g in got.items():
        r = ref[n]
        assert (g - r).abs().max().item() <= 1e-4 * r.abs().max().item(), n


# ------------------------------------------------------------------ GRU (FO + BPPSA backward)
def test_gru_gates_recompute_vs_oracle(lib):
    """bppsa_gru_gates (FO) against the oracle's gru_gates64 on the same
    fp32 h (gates are O(1): 1e-5 absolute)."""
    from oracle import bp
    from paper_1907_10134_b200 import api
    gw = W.gru_workload("M", 16, seed=4)
    p, tape = gw.params, gw.tape
    h0 = np.random.default_rng(1).standard_normal((16, 20)).astype(np.float32) * 0.2
    for hi in (None, h0):
        ref = bp.gru_gates64(gw.x, tape["h"], p, h_init=hi)
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        got = api.gru_gates(cu(gw.x), cu(tape["h"]), cu(p["W_ih3"]), cu(p["W_hh3"]), cu(p["b_ih3"]), cu(p["b_hh3"]),
                            h_init=None if hi is None else cu(hi))
        torch.cuda.synchronize()
        for k in ("h_prev", "r", "z", "n", "M"):
            assert np.abs(got[k].cpu().numpy() - ref[k]).max() < 1e-5, k


@pytest.mark.parametrize("F,C,B", [(259, 38, 16), (1034, 12, 64)])
def test_gru_bppsa_gradients_equal_autograd(lib, F, C, B):
    """cuDNN GRU forward + FO + BPPSA backward: every GRU parameter gradient
    within 1e-4 (max-norm relative) of torch autograd's."""
    from paper_1907_10134_b200.train import BppsaGruTrainer, IrmasGru
    torch.backends.cudnn.allow_tf32 = False
    torch.manual_seed(7)
    m = IrmasGru(C).cuda()
    x, y = W.irmas_like(F, C, B, 3)
    x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    _, logits = m(x)
    torch.nn.functional.cross_entropy(logits, y).backward()
    ref = {n: p.grad.clone() for n, p in m.rnn.named_parameters()}
    t = BppsaGruTrainer(m, lr=0.0)
    t.step(x, y)
    for n, p in m.rnn.named_parameters():
        e = ((p.grad - ref[n]).abs().max() / ref[n].abs().max()).item()
        assert e <= 1e-4, (n, e)


def test_gru_bppsa_training_matches_autograd(lib):
    from paper_1907_10134_b200.train import AutogradTrainer, BppsaGruTrainer, IrmasGru
    torch.backends.cudnn.allow_tf32 = False
    torch.manual_seed(0)
    ma = IrmasGru(24).cuda()
    mb = copy.deepcopy(ma)
    mb.rnn.flatten_parameters()
    ta, tb = BppsaGruTrainer(ma, lr=3e-4), AutogradTrainer(mb, lr=3e-4)
    la, lb = [], []
    for it in range(20):
        x, y = W.irmas_like(517, 24, 16, 50 + it)
        x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        la.append(ta.step(x, y))
        lb.append(tb.step(x, y))
    la, lb = np.array(la), np.array(lb)
    assert abs(la[0] - lb[0]) <= 1e-6 * abs(lb[0])
    assert np.abs(la - lb).max() <= 1e-3 * np.abs(lb).max(), (la, lb)
