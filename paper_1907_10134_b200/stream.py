"""Host-input BPPSA backward with the input copy overlapped (single GPU).

The inputs of a long sequence (h is 4.3 GB at config 4) take longer to cross
PCIe than the backward takes to run, so the backward is started on the part of
the sequence that has arrived.  The sequence is cut into G contiguous time
chunks — the multi-GPU shards of dist.py, on one device — and copied from
pinned host memory on a copy stream in REVERSE time order (the chunk holding
t = T-1 and the seed first).  Chunk r is scanned as soon as it lands:

  bppsa_scan_shard_up(r)      its leaves folded to one aggregate per sample
  bppsa_scan_shard_down(r)    its carry M_{r+1} ... M_{G-2} V from the
                              aggregates of the later chunks, all already
                              computed (reverse order), then its walk

so by the time the last chunk (t = 0) arrives only its own up/down sweep and
the weight gradients (bppsa_weight_grads_rnn over the whole sequence) remain.
Every step runs in libbppsa's kernels; this module only orders copies and
launches on two streams (no torch arithmetic).  The association differs from
the one-shot scan by the chunk boundaries only (reading 13).
"""
from __future__ import annotations

import torch

from . import api
from .dist import shard_bounds


class StreamedRnnBackward:
    """Pre-allocated device buffers, workspaces and streams for one shape."""

    def __init__(self, T: int, B: int, H: int, I: int, chunks: int = 8, block0: int = 0, block: int = 0,
                 device=None):
        dev = torch.device(device or "cuda")
        self.T, self.B, self.H, self.I, self.G = T, B, H, I, chunks
        self.block0, self.block = block0, block
        self.bounds = shard_bounds(T, chunks)
        self.h = torch.empty((T, B, H), device=dev)
        self.x = torch.empty((T, B, I), device=dev)
        self.W = torch.empty((H, H), device=dev)
        self.seed = torch.empty((B, H), device=dev)
        self.grad = torch.empty((T, B, H), device=dev)
        self.grad_init = torch.empty((B, H), device=dev)
        self.aggs = torch.empty((chunks, B, H * H), device=dev)
        self.jacs = [api.jacobians_rnn(self.h[lo:hi], self.W) for lo, hi in self.bounds]
        self.ws = [api.workspace(api.scan_workspace_size(j, "blocked", block0, block), dev) for j in self.jacs]
        self.ws_w = api.workspace(api.weight_grads_workspace_size(T, B, H, I), dev)
        self.out = (torch.empty((H, I), device=dev), torch.empty((H, H), device=dev), torch.empty((H,), device=dev))
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.events = [torch.cuda.Event() for _ in range(chunks + 1)]

    def run(self, h_host: torch.Tensor, x_host: torch.Tensor, W_host: torch.Tensor, seed_host: torch.Tensor,
            out_host=None):
        """Backward from pinned host inputs; returns device (dW_ih, dW_hh, db,
        grad_h, dl/dh_init), or copies (dW_ih, dW_hh, db, dl/dh_init) into the
        pinned `out_host` tensors when given.  Enqueued on the current stream."""
        cs, cur = self.copy_stream, torch.cuda.current_stream()
        G = self.G
        cs.wait_stream(cur)                      # buffers are free once earlier work on `cur` is done
        with torch.cuda.stream(cs):
            self.W.copy_(W_host, non_blocking=True)
            self.seed.copy_(seed_host, non_blocking=True)
            for k, r in enumerate(reversed(range(G))):
                lo, hi = self.bounds[r]
                self.h[lo:hi].copy_(h_host[lo:hi], non_blocking=True)
                self.events[k].record(cs)
            self.x.copy_(x_host, non_blocking=True)
            self.events[G].record(cs)
        for k, r in enumerate(reversed(range(G))):
            cur.wait_event(self.events[k])
            head = r == G - 1
            seed = self.seed if head else None
            api.scan_shard_up(self.jacs[r], seed, self.aggs[r], self.ws[r], self.block0, self.block)
            lo, hi = self.bounds[r]
            api.scan_shard_down(self.jacs[r], seed, None if head else self.aggs, r, G, self.grad[lo:hi],
                                self.grad_init if r == 0 else None, self.ws[r], self.block0, self.block)
        cur.wait_event(self.events[G])
        dWih, dWhh, db = api.weight_grads_rnn(self.x, self.h, self.grad, ws=self.ws_w, out=self.out)
        if out_host is not None:
            for o, s in zip(out_host, (dWih, dWhh, db, self.grad_init)):
                o.copy_(s, non_blocking=True)
        return dWih, dWhh, db, self.grad, self.grad_init
