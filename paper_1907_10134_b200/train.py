"""End-to-end RNN training with the BPPSA backward.

The paper trains a vanilla tanh RNN on synthetic bitstreams (P:303-317:
x_t ~ Bernoulli(0.05 + 0.1 c), the class c read from h_{T-1} by a linear
head, softmax cross-entropy) and reports the loss against wall-clock time
for BPPSA and for plain back-propagation (the 2.73x end-to-end
claim).  One iteration here is

  forward   torch nn.RNN (cuDNN) -> h_0..h_{T-1}; the head on h_{T-1}
  backward  the head by autograd (it is not part of the scan) -> seed dl/dh_{T-1};
            bppsa_scan over the RNN leaves -> every dl/dh_t;
            bppsa_weight_grads_rnn -> dW_ih, dW_hh, db (= db_ih = db_hh, reading 9)
  update    torch.optim.Adam

and `step_autograd` is the same iteration with torch's own backward (cuDNN),
the baseline.  Only the backward differs: the two trainers see the same
forward, the same optimizer and the same data.
"""
from __future__ import annotations

import torch

from . import api


class BitstreamRnn(torch.nn.Module):
    """nn.RNN(I, H, tanh) + Linear(H, classes) on the last hidden state."""

    def __init__(self, H: int = 20, I: int = 1, classes: int = 10):
        super().__init__()
        self.rnn = torch.nn.RNN(I, H, nonlinearity="tanh")
        self.head = torch.nn.Linear(H, classes)

    def forward(self, x):
        h, _ = self.rnn(x)                     # [T, B, H], h_0 = 0 (reading 7)
        return h, self.head(h[-1])


class BppsaTrainer:
    """One training iteration with the BPPSA backward (buffers kept per shape)."""

    def __init__(self, model: BitstreamRnn, lr: float, block0: int = 0, block: int = 0):
        self.model, self.block0, self.block = model, block0, block
        self.opt = torch.optim.Adam(model.parameters(), lr=lr)
        self._shape = None

    def _buffers(self, T, B, H, I, dev):
        if self._shape != (T, B, H, I):
            self.grad = torch.empty((T, B, H), device=dev)
            self.ws_w = api.workspace(api.weight_grads_workspace_size(T, B, H, I), dev)
            self.ws = None
            self._shape = (T, B, H, I)

    def step(self, x: torch.Tensor, labels: torch.Tensor) -> float:
        m = self.model
        T, B, I = x.shape
        H = m.rnn.hidden_size
        self._buffers(T, B, H, I, x.device)
        self.opt.zero_grad(set_to_none=True)
        with torch.no_grad():
            h, _ = m.rnn(x)
        h = h.contiguous()
        # the head by autograd: its parameter gradients and the seed dl/dh_{T-1}
        hl = h[-1].detach().requires_grad_(True)
        loss = torch.nn.functional.cross_entropy(m.head(hl), labels)
        loss.backward()
        seed = hl.grad.contiguous()
        W_hh = m.rnn.weight_hh_l0.detach().contiguous()
        jac = api.jacobians_rnn(h, W_hh)
        if self.ws is None:
            self.ws = api.workspace(api.scan_workspace_size(jac, "blocked", self.block0, self.block), x.device)
        api.scan(jac, seed, grad_h=self.grad, ws=self.ws, block0=self.block0, block=self.block)
        dWih, dWhh, db = api.weight_grads_rnn(x.contiguous(), h, self.grad, ws=self.ws_w)
        m.rnn.weight_ih_l0.grad = dWih
        m.rnn.weight_hh_l0.grad = dWhh
        m.rnn.bias_ih_l0.grad = db
        m.rnn.bias_hh_l0.grad = db.clone()
        self.opt.step()
        return float(loss.detach())


class IrmasGru(torch.nn.Module):
    """The paper's GRU model: nn.GRU(C, H) + Linear(H, classes)
    on the last hidden state (H = 20, 11 classes: reading 21)."""

    def __init__(self, C: int, H: int = 20, classes: int = 11):
        super().__init__()
        self.rnn = torch.nn.GRU(C, H)
        self.head = torch.nn.Linear(H, classes)

    def forward(self, x):
        h, _ = self.rnn(x)
        return h, self.head(h[-1])


class BppsaGruTrainer:
    """GRU training with the BPPSA backward: cuDNN forward (gates hidden), the
    gate recompute "FO" (bppsa_gru_gates), the eqn:gru_jcb leaves,
    the scan, the GRU weight gradients, Adam (lr 3e-4 in the paper's runs)."""

    def __init__(self, model: IrmasGru, lr: float, block0: int = 0, block: int = 0):
        self.model, self.block0, self.block = model, block0, block
        self.opt = torch.optim.Adam(model.parameters(), lr=lr)
        self._shape = None

    def step(self, x: torch.Tensor, labels: torch.Tensor) -> float:
        m = self.model
        T, B, I = x.shape
        H = m.rnn.hidden_size
        if self._shape != (T, B, H, I):
            self.grad = torch.empty((T, B, H), device=x.device)
            self.ws_w = api.workspace(api.weight_grads_workspace_size(T, B, H, I), x.device)
            self.ws = None
            self._shape = (T, B, H, I)
        self.opt.zero_grad(set_to_none=True)
        with torch.no_grad():
            h, _ = m.rnn(x)
        h = h.contiguous()
        hl = h[-1].detach().requires_grad_(True)
        loss = torch.nn.functional.cross_entropy(m.head(hl), labels)
        loss.backward()
        seed = hl.grad.contiguous()
        r = m.rnn
        W_hh3 = r.weight_hh_l0.detach().contiguous()
        xc = x.contiguous()
        tape = api.gru_gates(xc, h, r.weight_ih_l0.detach().contiguous(), W_hh3, r.bias_ih_l0.detach().contiguous(),
                             r.bias_hh_l0.detach().contiguous())
        jac = api.jacobians_gru(tape["h_prev"], tape["r"], tape["z"], tape["n"], tape["M"], W_hh3)
        if self.ws is None:
            self.ws = api.workspace(api.scan_workspace_size(jac, "blocked", self.block0, self.block), x.device)
        api.scan(jac, seed, grad_h=self.grad, ws=self.ws, block0=self.block0, block=self.block)
        dWih, dWhh, dbih, dbhh = api.weight_grads_gru(xc, tape, self.grad, ws=self.ws_w)
        r.weight_ih_l0.grad, r.weight_hh_l0.grad = dWih, dWhh
        r.bias_ih_l0.grad, r.bias_hh_l0.grad = dbih, dbhh
        self.opt.step()
        return float(loss.detach())


class AutogradTrainer:
    """The baseline: the same iteration with torch's backward (cuDNN)."""

    def __init__(self, model: BitstreamRnn, lr: float):
        self.model = model
        self.opt = torch.optim.Adam(model.parameters(), lr=lr)

    def step(self, x: torch.Tensor, labels: torch.Tensor) -> float:
        self.opt.zero_grad(set_to_none=True)
        _, logits = self.model(x)
        loss = torch.nn.functional.cross_entropy(logits, labels)
        loss.backward()
        self.opt.step()
        return float(loss.detach())
