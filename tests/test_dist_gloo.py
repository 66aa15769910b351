"""Multi-process (gloo, CPU) tests of the contiguous-time-shard protocol of
paper_1907_10134_b200.dist: shard bounds, head rank, aggregate
layout, the all-gather and the carry order.  The per-rank arithmetic is the
oracle's (tests only); on the GPU the same protocol drives
bppsa_scan_shard_up / _down (tests/test_gpu_parity.py::test_shard_loopback)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bp, scan as S


class OracleShardBackend:
    """The dist protocol's backend interface implemented with the oracle, using
    the library's aggregate layout ([B, H*H] column-major; the head rank's
    vector in the first H floats)."""

    def __init__(self, JT, lo, hi):
        self.JT, self.lo, self.hi = JT, lo, hi
        self.B, self.H = JT.shape[1], JT.shape[2]

    def up(self, seed):
        el = S.shard_aggregate(self.JT, self.lo, self.hi, None if seed is None else seed.numpy())
        out = np.zeros((self.B, self.H * self.H))
        if el.kind == "v":
            out[:, :self.H] = el.val
        else:
            out[:] = el.val.transpose(0, 2, 1).reshape(self.B, -1)     # column-major
        return torch.from_numpy(out)

    def down(self, seed, gathered, rank, world, grad_h=None, want_init=False):
        if gathered is None:                       # head: carry = seed
            carry = seed.numpy()
        else:
            G = gathered.numpy()
            aggs = [S.El("m", G[r].reshape(self.B, self.H, self.H).transpose(0, 2, 1)) for r in range(world)]
            aggs[world - 1] = S.El("v", G[world - 1][:, :self.H])
            carry = S.shard_carries(aggs)[rank]
        out, init = S.shard_local_grads(self.JT, self.lo, self.hi, carry)
        return torch.from_numpy(out), torch.from_numpy(init)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, T, B, H, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1907_10134_b200.dist import sharded_scan, shard_bounds
        rng = np.random.default_rng(1234)          # same inputs on every rank
        JT = rng.standard_normal((T, B, H, H)) * 0.4
        g = rng.standard_normal((B, H))
        lo, hi = shard_bounds(T, world)[rank]
        be = OracleShardBackend(JT, lo, hi)
        seed = torch.from_numpy(g) if rank == world - 1 else None
        grad, init = sharded_scan(be, seed)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, grad.numpy(), init.numpy()))
        if rank == 0:
            ref, ref_init = bp.bp_dense(JT, g)
            got = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
            q.put((float(np.abs(got - ref).max() / np.abs(ref).max()),
                   float(np.abs(parts[0][3] - ref_init).max() / np.abs(ref).max())))
        # the seed must be given by exactly the last rank (every rank wrong here,
        # so each one must refuse before entering the collective)
        bad = None if rank == world - 1 else torch.from_numpy(g)
        try:
            sharded_scan(be, bad)
            ok = world == 1
        except ValueError:
            ok = True
        dist.all_gather_object(parts, ok)
        if rank == 0:
            q.put(all(parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 50), (3, 31), (4, 64)])
def test_sharded_protocol_gloo(world, T):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, 2, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    err, err_init = q.get(timeout=5)
    assert err < 1e-12 and err_init < 1e-12
    assert q.get(timeout=5)


def test_shard_bounds():
    from paper_1907_10134_b200.dist import shard_bounds
    for T in (8, 9, 1000, 1 << 20):
        for G in (1, 2, 3, 8):
            b = shard_bounds(T, G)
            assert b[0][0] == 0 and b[-1][1] == T
            assert all(b[i][1] == b[i + 1][0] for i in range(G - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1
    with pytest.raises(ValueError):
        shard_bounds(3, 4)
