"""Multi-GPU BPPSA: contiguous time shards, one exchange.

Rank order = time order; rank r owns t in [lo_r, hi_r) and the last rank holds
t = T-1 and the seed (the "head" shard, first in scan order).  Protocol:

  1. local leaf + up-sweep to one aggregate per sample        (bppsa_scan_shard_up)
       rank < G-1:  M_r = J_lo^T ... J_{hi-1}^T   [B, H*H] column-major
       rank = G-1:  V   = grad_h[lo-1]            [B, H] in the first H floats
  2. all-gather of the aggregates over NCCL (torch.distributed; NVLink on the
     8xB200 box) — the only data-path collective; or, with a PeerExchange,
     P2P stores into every rank's mailbox from the up-sweep's own top-level
     kernel (bppsa_scan_shard_up_publish) and a flag wait — no NCCL
  3. carry for rank r: M_{r+1} ... M_{G-2} V and the local down-sweep on the
     device                                                     (bppsa_scan_shard_down)
  4. (caller) all-reduce of the weight gradients.

The protocol is written against a small backend interface so the host logic
can be exercised with the gloo backend on CPU (tests/test_dist_gloo.py plugs in
an oracle-backed backend); the product backend is `CudaShardBackend`.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(T: int, G: int):
    """Contiguous shards in time order, remainder spread over the first ranks."""
    if T < G:
        raise ValueError("need at least one step per rank")
    base, rem = divmod(T, G)
    out, lo = [], 0
    for r in range(G):
        sz = base + (1 if r < rem else 0)
        out.append((lo, lo + sz))
        lo += sz
    return out


class CudaShardBackend:
    """bppsa_scan_shard_up / _down on this rank's GPU (workspace kept between)."""

    def __init__(self, jac, block0: int = 0, block: int = 0):
        from . import api
        self.api, self.jac, self.block0, self.block = api, jac, block0, block
        self.ws = api.workspace(api.scan_workspace_size(jac, "blocked", block0, block))

    def up(self, seed):
        B, H = self.jac.B, self.jac.H
        agg = torch.empty((B, H * H), dtype=torch.float32, device="cuda")
        self.api.scan_shard_up(self.jac, seed, agg, self.ws, self.block0, self.block)
        return agg

    def up_publish(self, seed, ex: "PeerExchange"):
        """The up-sweep with the peer-memory publish fused into its top level
        (bppsa_scan_shard_up_publish) for epoch ex.epoch."""
        B, H = self.jac.B, self.jac.H
        agg = torch.empty((B, H * H), dtype=torch.float32, device="cuda")
        self.api.scan_shard_up_publish(self.jac, seed, agg, self.ws, ex.rank, ex.world, ex.mail_ptrs, ex.flag_ptrs,
                                       ex.counter, ex.acks, ex.epoch, self.block0, self.block)
        return agg

    def down(self, seed, gathered, rank, world, grad_h=None, want_init=False):
        T, B, H = self.jac.T, self.jac.B, self.jac.H
        if grad_h is None:
            grad_h = torch.empty((T, B, H), dtype=torch.float32, device="cuda")
        gi = torch.empty((B, H), dtype=torch.float32, device="cuda") if want_init else None
        self.api.scan_shard_down(self.jac, seed, gathered, rank, world, grad_h, gi, self.ws,
                                 self.block0, self.block)
        return grad_h, gi


class PeerExchange:
    """The carry exchange over peer memory (bppsa_exchange_publish / _wait)
    instead of an NCCL all-gather: this rank's mailbox [2][world][B][H*H] and
    flags [world] are mapped into every other rank with CUDA IPC (handles
    swapped once through torch.distributed), so the up-sweep aggregate is
    stored straight into every peer's memory over NVLink and the down-sweep
    waits on the flags of the later ranks only.  Back-pressure: after its
    down-sweep read the mailbox, a rank acks the epoch in every later rank
    (`release`), and a writer publishing epoch e first waits for the acks of
    e - 2 (whose slot it overwrites).  One instance per (rank, shape); every
    call of `exchange` is a new epoch, followed by one `release`."""

    def __init__(self, B: int, H: int, group=None):
        from torch.multiprocessing.reductions import reduce_tensor
        from . import api
        self.api, self.group = api, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.n = B * H * H
        self.mail = torch.zeros((2, self.world, B, H * H), dtype=torch.float32, device="cuda")
        self.flags = torch.zeros(self.world, dtype=torch.int32, device="cuda")
        self.acks = torch.zeros(self.world, dtype=torch.int32, device="cuda")
        self.counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        mine = (self.rank, reduce_tensor(self.mail), reduce_tensor(self.flags), reduce_tensor(self.acks))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._peers = []                                   # keep the mappings alive
        mail_ptrs, flag_ptrs, ack_ptrs = [0] * self.world, [0] * self.world, [0] * self.world
        for r, (fm, am), (ff, af), (fa, aa) in allh:
            if r == self.rank:
                m, f, k = self.mail, self.flags, self.acks
            else:
                m, f, k = fm(*am), ff(*af), fa(*aa)
                self._peers.append((m, f, k))
            mail_ptrs[r], flag_ptrs[r], ack_ptrs[r] = m.data_ptr(), f.data_ptr(), k.data_ptr()
        self.mail_ptrs = torch.tensor(mail_ptrs, dtype=torch.int64, device="cuda")
        self.flag_ptrs = torch.tensor(flag_ptrs, dtype=torch.int64, device="cuda")
        self.ack_ptrs = torch.tensor(ack_ptrs, dtype=torch.int64, device="cuda")
        self.epoch = 0
        dist.barrier(group=group)

    def up_and_exchange(self, backend, seed) -> torch.Tensor:
        """The fused form: the backend's up-sweep publishes into the mailboxes
        from its own top-level kernel (no separate publish launch), then the
        wait; returns the gathered view like `exchange`."""
        self.epoch += 1
        backend.up_publish(seed, self)
        self.api.exchange_wait(self.flags, self.rank, self.world, self.epoch)
        return self.mail[self.epoch & 1]

    def exchange(self, agg: torch.Tensor) -> torch.Tensor:
        """Publish this rank's aggregate, wait for the later ranks'; returns the
        gathered [world, B, H*H] view (valid for kernels after this call)."""
        self.epoch += 1
        self.api.exchange_publish(agg.contiguous(), self.rank, self.world, self.mail_ptrs, self.flag_ptrs,
                                  self.counter, self.acks, self.epoch)
        self.api.exchange_wait(self.flags, self.rank, self.world, self.epoch)
        return self.mail[self.epoch & 1]

    def release(self):
        """This rank's reads of the current epoch's mailbox are enqueued: ack it."""
        self.api.exchange_ack(self.rank, self.world, self.ack_ptrs, self.epoch)


def sharded_scan(backend, seed, group=None, want_init: bool = False, grad_h=None, exchange=None, fused: bool = True):
    """Run the 3-step protocol on this rank.  `seed` must be given on the last
    rank only (it holds t = T-1).  Returns (local grad_h, J_lo^T grad_h[lo])."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    head = rank == world - 1
    if head != (seed is not None):
        raise ValueError("exactly the last rank passes the seed")
    if world > 1 and exchange is not None and fused and hasattr(backend, "up_publish"):
        # peer-memory exchange fused into the up-sweep's top level (no NCCL, no publish launch)
        gathered = exchange.up_and_exchange(backend, seed).view(world, backend.jac.B, backend.jac.H ** 2)
    elif world > 1 and exchange is not None:             # peer-memory exchange (no NCCL)
        agg = backend.up(seed)
        gathered = exchange.exchange(agg).view((world,) + tuple(agg.shape))
    elif world > 1:
        agg = backend.up(seed)
        flat = torch.empty((world * agg.shape[0],) + tuple(agg.shape[1:]), dtype=agg.dtype, device=agg.device)
        dist.all_gather_into_tensor(flat, agg.contiguous(), group=group)    # concat form (NCCL and gloo)
        gathered = flat.view((world,) + tuple(agg.shape))
    else:
        gathered = backend.up(seed).unsqueeze(0)
    out = backend.down(seed, None if head else gathered, rank, world, grad_h=grad_h, want_init=want_init)
    if world > 1 and exchange is not None:
        exchange.release()
    return out
