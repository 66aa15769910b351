"""Config 5: the transposed-Jacobian chain of a VGG-style conv
stack, assembled through the library's analytical CSR builders (Algs. 2-10):
host patterns from bppsa_csr_*_pattern, device data from bppsa_csr_*_data.
Marshalling only — every value is produced by libbppsa.
"""
from __future__ import annotations

import numpy as np
import torch

from . import api


def conv_stack_ops(cfg, in_ch: int = 3, hw: int = 32):
    """[('conv', ci, co, h, w) | ('relu', c, h, w) | ('pool', c, h, w)] with the
    operator's input spatial size (VGG-11 cfg: 64, M, 128, M, 256, 256, M, ...)."""
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


class CsrChain:
    """Patterns (host) and data (device) of J_1^T .. J_n^T for one batch.

    weights: per conv layer [co, ci, 3, 3] (numpy; pruned taps are zeros and
    leave the pattern); relu_in: per ReLU [B, c, h, w] (device tensors, the
    ReLU inputs); pool_idx: per max-pool [B, c, h/2, w/2] int64 (device)."""

    def __init__(self, cfg, weights, relu_in, pool_idx, hw: int = 32, in_ch: int = 3):
        self.ops = conv_stack_ops(cfg, in_ch, hw)
        self.patterns, self.data, self.batched = [], [], []
        wi = ri = pi = 0
        for op in self.ops:
            if op[0] == "conv":
                _, ci, co, h, w = op
                wt = np.ascontiguousarray(weights[wi], dtype=np.float32)
                ip, ix, tap = api.csr_conv3x3_pattern(ci, co, h, w, wt, drop_zero=True)
                self.patterns.append((ci * h * w, co * h * w, ip, ix))
                wdev = torch.from_numpy(wt.reshape(-1)).cuda()
                self.data.append(api.csr_conv_data(torch.from_numpy(tap).cuda(), wdev))
                self.batched.append(0)
                wi += 1
            elif op[0] == "relu":
                _, c, h, w = op
                d = c * h * w
                self.patterns.append((d, d, np.arange(d + 1, dtype=np.int64), np.arange(d, dtype=np.int32)))
                x = relu_in[ri].reshape(relu_in[ri].shape[0], -1).contiguous()
                self.data.append(api.csr_relu_data(x))
                self.batched.append(1)
                ri += 1
            else:
                _, c, h, w = op
                ip, ix = api.csr_maxpool_pattern(c, h, w)
                self.patterns.append((c * h * w, c * (h // 2) * (w // 2), ip, ix))
                self.data.append(api.csr_maxpool_data(pool_idx[pi].contiguous(), c, h, w))
                self.batched.append(1)
                pi += 1
        self.n = len(self.ops)

    def plan(self, up_levels: int, down_levels: int, max_contributions: int = 0) -> api.CsrPlan:
        return api.csr_plan_create(self.patterns, up_levels, down_levels, max_contributions)
