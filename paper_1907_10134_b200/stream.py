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
launches on two streams (no torch arithmetic).  When the chunks are whole
parts of the tensor-core weight gradients, those run chunk by chunk too
(bppsa_weight_grads_rnn_rows, one chunk behind: a chunk's first h_prev is the
last h row of the chunk before it, which arrives next), so only the last
chunk's share and the fixed-order reduction remain after the last copy;
the result is bit-identical to one bppsa_weight_grads_rnn call.  The association differs from
the one-shot scan by the chunk boundaries only (reading 13).
"""
from __future__ import annotations

import torch

from . import api
from .dist import shard_bounds


class StreamedRnnBackward:
    """Pre-allocated device buffers, workspaces and streams for one shape."""

    def __init__(self, T: int, B: int, H: int, I: int, chunks: int = 8, block0: int = 0, block: int = 0,
                 device=None, tail: int = 0):
        dev = torch.device(device or "cuda")
        self.T, self.B, self.H, self.I = T, B, H, I
        self.block0, self.block = block0, block
        bounds = shard_bounds(T, chunks)
        # tail > 0: the chunk holding t = 0 (the last to arrive) is cut into
        # tail + 1 pieces of 1/2^tail, 1/2^tail, 1/2^(tail-1), ..., 1/2 of it, so
        # only a small piece's sweep is left after the last copy (measured at
        # C4: 86.5 vs 82.5 ms — a shard's sweep has a latency floor of one
        # block's dependent steps, so small shards only add serial work; off by
        # default)
        lo0, hi0 = bounds[0]
        c = hi0 - lo0
        if tail > 0 and c % (1 << tail) == 0:
            cuts, sz, pos = [], c >> tail, lo0
            for k in range(tail + 1):
                step = sz if k == 0 else sz << (k - 1)
                cuts.append((pos, pos + step))
                pos += step
            bounds = cuts + bounds[1:]
        self.bounds = bounds
        self.G = chunks = len(bounds)
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
        # weight gradients chunk by chunk as each chunk's grad_h is final, when
        # the chunks are whole parts of the tensor-core path (bit-identical to
        # one call over the sequence); else one call at the end
        pr = api.weight_grads_rnn_part_rows(T, B, H, I)
        self.wg_rows = pr > 0 and all((lo * B) % pr == 0 for lo, _ in self.bounds)
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
                if self.wg_rows:
                    self.x[lo:hi].copy_(x_host[lo:hi], non_blocking=True)
                self.events[k].record(cs)
            if not self.wg_rows:
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
            if self.wg_rows and r + 1 < G:
                # the later chunk's rows: its grad_h is final and its first h_prev
                # (the last h row of chunk r) has just arrived
                lo1, hi1 = self.bounds[r + 1]
                api.weight_grads_rnn_rows(self.x, self.h, self.grad, lo1 * self.B, hi1 * self.B, self.ws_w)
        cur.wait_event(self.events[G])
        if self.wg_rows:
            lo0, hi0 = self.bounds[0]                 # chunk 0: h_prev of t = 0 is h_init (0)
            api.weight_grads_rnn_rows(self.x, self.h, self.grad, lo0 * self.B, hi0 * self.B, self.ws_w)
            dWih, dWhh, db = api.weight_grads_rnn_reduce(self.T, self.B, self.H, self.I, self.ws_w, out=self.out)
        else:
            dWih, dWhh, db = api.weight_grads_rnn(self.x, self.h, self.grad, ws=self.ws_w, out=self.out)
        if out_host is not None:
            for o, s in zip(out_host, (dWih, dWhh, db, self.grad_init)):
                o.copy_(s, non_blocking=True)
        return dWih, dWhh, db, self.grad, self.grad_init
