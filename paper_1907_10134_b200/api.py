"""Thin Python binding of libbppsa.so (include/bppsa.h) — argument marshalling
only.  Every arithmetic step of the path runs in the library's sm_100a
kernels; torch supplies device memory, the current CUDA stream and (for the
sharded scan) the NCCL process group.  There is no CPU fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbppsa.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
_lib = C.CDLL(_LIB_PATH)

# ----------------------------------------------------------------- ABI types
OK = 0
JAC_DENSE, JAC_RNN_TANH, JAC_GRU = 0, 1, 2
SCAN_BLOCKED, SCAN_ALG1, SCAN_LINEAR, SCAN_HYBRID = 0, 1, 2, 3
MODES = {"blocked": SCAN_BLOCKED, "alg1": SCAN_ALG1, "linear": SCAN_LINEAR, "hybrid": SCAN_HYBRID}

_vp, _i, _sz = C.c_void_p, C.c_int, C.c_size_t


class _Jac(C.Structure):
    _fields_ = [("kind", _i), ("T", _i), ("B", _i), ("H", _i), ("JT", _vp), ("h", _vp), ("W_hh", _vp),
                ("h_prev", _vp), ("r", _vp), ("z", _vp), ("n", _vp), ("M", _vp), ("W_hh3", _vp)]


class _Opts(C.Structure):
    _fields_ = [("mode", _i), ("block0", _i), ("block", _i), ("leaf_impl", _i), ("events", C.POINTER(_vp)),
                ("n_events", _i), ("launches", C.POINTER(_i)), ("up_levels", _i), ("down_levels", _i)]


EXPORTS = {
    "bppsa_status_str": (C.c_char_p, [_i]),
    "bppsa_last_error": (C.c_char_p, []),
    "bppsa_version": (_i, []),
    "bppsa_jacobians_rnn": (_i, [_i, _i, _i, _vp, _vp, _vp, C.POINTER(_Jac), _vp]),
    "bppsa_jacobians_gru": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_Jac), _vp]),
    "bppsa_scan_workspace_size": (_i, [C.POINTER(_Jac), C.POINTER(_Opts), C.POINTER(_sz)]),
    "bppsa_scan": (_i, [C.POINTER(_Jac), _vp, _vp, _vp, _vp, _sz, C.POINTER(_Opts), _vp]),
    "bppsa_weight_grads_rnn_part_rows": (_i, [_i, _i, _i, _i, C.POINTER(C.c_longlong)]),
    "bppsa_weight_grads_rnn_rows": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, C.c_longlong, C.c_longlong, _vp, _sz,
                                         _vp]),
    "bppsa_weight_grads_rnn_reduce": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _sz, _vp]),
    "bppsa_exchange_publish": (_i, [_vp, C.c_longlong, _i, _i, _vp, _vp, _vp, _vp, C.c_uint, _vp]),
    "bppsa_exchange_ack": (_i, [_i, _i, _vp, C.c_uint, _vp]),
    "bppsa_exchange_wait": (_i, [_vp, _i, _i, C.c_uint, _vp]),
    "bppsa_gru_gates": (_i, [_i, _i, _i, _i] + [_vp] * 12 + [_vp]),
    "bppsa_scan_affine": (_i, [C.POINTER(_Jac), _vp, _vp, _vp, _vp, _vp, _sz, C.POINTER(_Opts), _vp]),
    "bppsa_scan_shard_up": (_i, [C.POINTER(_Jac), _vp, _vp, _vp, _sz, C.POINTER(_Opts), _vp]),
    "bppsa_scan_shard_up_publish": (_i, [C.POINTER(_Jac), _vp, _vp, _vp, _sz, C.POINTER(_Opts), _i, _i, _vp, _vp,
                                         _vp, _vp, C.c_uint, _vp]),
    "bppsa_scan_shard_down": (_i, [C.POINTER(_Jac), _vp, _vp, _i, _i, _vp, _vp, _vp, _sz, C.POINTER(_Opts), _vp]),
    "bppsa_weight_grads_workspace_size": (_i, [_i, _i, _i, _i, C.POINTER(_sz)]),
    "bppsa_weight_grads_rnn": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "bppsa_weight_grads_gru": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _sz, _vp]),
}

class _CsrPat(C.Structure):
    _fields_ = [("rows", _i), ("cols", _i), ("nnz", C.c_longlong), ("indptr", _vp), ("indices", _vp)]


_ll, _pp = C.c_longlong, C.POINTER(_vp)
EXPORTS.update({
    "bppsa_csr_plan_create": (_i, [C.POINTER(_CsrPat), _i, _i, _i, _ll, C.POINTER(_vp)]),
    "bppsa_csr_plan_create_symbolic": (_i, [C.POINTER(_CsrPat), _i, _i, _i, C.POINTER(_vp)]),
    "bppsa_csr_plan_destroy": (None, [_vp]),
    "bppsa_csr_plan_workspace_size": (_i, [_vp, _i, C.POINTER(_i), C.POINTER(_sz)]),
    "bppsa_csr_plan_info": (_i, [_vp, C.POINTER(_ll), C.POINTER(_ll), C.POINTER(_i)]),
    "bppsa_csr_scan": (_i, [_vp, _i, _pp, C.POINTER(_i), _vp, _pp, _vp, _sz, _vp]),
    "bppsa_csr_conv3x3_pattern": (_i, [_i, _i, _i, _i, _vp, _i, C.POINTER(_ll), _vp, _vp, _vp]),
    "bppsa_csr_conv_data": (_i, [_ll, _vp, _vp, _vp, _vp]),
    "bppsa_csr_relu_data": (_i, [_ll, _i, _vp, _vp, _vp]),
    "bppsa_csr_maxpool_pattern": (_i, [_i, _i, _i, _vp, _vp]),
    "bppsa_csr_maxpool_data": (_i, [_i, _i, _i, _i, _vp, _vp, _vp]),
    "bppsa_csr_plan_steps": (_i, [_vp, _vp, _i, C.POINTER(_i)]),
    "bppsa_csr_conv3x3_build_size": (_i, [_i, _i, _i, _i, _i, C.POINTER(_ll), C.POINTER(_sz)]),
    "bppsa_csr_conv3x3_build": (_i, [_i, _i, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "bppsa_csr_maxpool_build": (_i, [_i, _i, _i, _vp, _vp, _vp]),
    "bppsa_csr_identity_build": (_i, [_ll, _vp, _vp, _vp]),
})


class _CsrStep(C.Structure):
    _fields_ = [("kind", _i), ("phase", _i), ("level", _i), ("critical", _i), ("flops", _ll),
                ("dense_flops", _ll)]


STEP_KIND = ("mm", "mv")
STEP_PHASE = ("up", "bridge", "down", "extra", "bp")
for _name, (_res, _args) in EXPORTS.items():
    _f = getattr(_lib, _name)
    _f.restype, _f.argtypes = _res, _args


class BppsaError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.bppsa_status_str(status).decode()
        detail = _lib.bppsa_last_error().decode()
        super().__init__(f"{where}: {msg}: {detail}")
        self.status = status


def _check(status: int, where: str) -> None:
    if status != OK:
        raise BppsaError(status, where)


def _ptr(t: torch.Tensor | None, name: str = "tensor"):
    if t is None:
        return None
    if not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    return t.data_ptr()


def _req(t: torch.Tensor | None, shape: tuple, name: str, dev: torch.device | None = None) -> None:
    """Shape / device check of a caller tensor before its raw pointer crosses
    the C ABI (the library cannot see extents: a wrong-shaped buffer would be
    read or written out of bounds)."""
    if t is None:
        return
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch.Tensor")
    if tuple(t.shape) != tuple(int(v) for v in shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if dev is not None and t.device != dev:
        raise ValueError(f"{name} is on {t.device}, expected {dev}")


def _ws(ws: torch.Tensor, dev: torch.device) -> None:
    if ws.dtype != torch.uint8 or not ws.is_cuda or not ws.is_contiguous() or ws.device != dev:
        raise ValueError(f"workspace must be a contiguous uint8 CUDA tensor on {dev}")


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def version() -> int:
    return _lib.bppsa_version()


# ----------------------------------------------------------------- leaves
class Jacobians:
    """A bppsa_jac descriptor plus references that keep its tensors alive."""

    def __init__(self, desc: _Jac, keep):
        self.desc = desc
        self._keep = keep

    T = property(lambda self: self.desc.T)
    B = property(lambda self: self.desc.B)
    H = property(lambda self: self.desc.H)
    kind = property(lambda self: self.desc.kind)


def jacobians_rnn(h: torch.Tensor, W_hh: torch.Tensor, JT_out: torch.Tensor | None = None, stream=None):
    """bppsa_jacobians_rnn: J_t^T = W_hh^T diag(1-h_t^2) (fused descriptor, or
    materialised into JT_out [T,B,H,H])."""
    if h.dim() != 3:
        raise ValueError("h must be [T, B, H]")
    T, B, H = h.shape
    _req(W_hh, (H, H), "W_hh", h.device)
    _req(JT_out, (T, B, H, H), "JT_out", h.device)
    d = _Jac()
    _check(_lib.bppsa_jacobians_rnn(T, B, H, _ptr(h, "h"), _ptr(W_hh, "W_hh"), _ptr(JT_out, "JT_out"),
                                    C.byref(d), _stream(stream)), "bppsa_jacobians_rnn")
    return Jacobians(d, (h, W_hh, JT_out))


def jacobians_gru(h_prev, r, z, n, M, W_hh3, JT_out: torch.Tensor | None = None, stream=None):
    """bppsa_jacobians_gru: eqn:gru_jcb leaves from the saved GRU tape."""
    if r.dim() != 3:
        raise ValueError("r must be [T, B, H]")
    T, B, H = r.shape
    for t_, nm in ((h_prev, "h_prev"), (z, "z"), (n, "n"), (M, "M")):
        _req(t_, (T, B, H), nm, r.device)
    _req(W_hh3, (3 * H, H), "W_hh3", r.device)
    _req(JT_out, (T, B, H, H), "JT_out", r.device)
    d = _Jac()
    _check(_lib.bppsa_jacobians_gru(T, B, H, _ptr(h_prev, "h_prev"), _ptr(r, "r"), _ptr(z, "z"), _ptr(n, "n"),
                                    _ptr(M, "M"), _ptr(W_hh3, "W_hh3"), _ptr(JT_out, "JT_out"), C.byref(d),
                                    _stream(stream)), "bppsa_jacobians_gru")
    return Jacobians(d, (h_prev, r, z, n, M, W_hh3, JT_out))


def jacobians_dense(JT: torch.Tensor) -> Jacobians:
    """A DENSE descriptor over caller-provided J_t^T [T,B,H,H] (row-major)."""
    if JT.dim() != 4 or JT.shape[2] != JT.shape[3]:
        raise ValueError("JT must be [T, B, H, H]")
    T, B, H, H2 = JT.shape
    d = _Jac()
    d.kind, d.T, d.B, d.H, d.JT = JAC_DENSE, T, B, H, _ptr(JT, "JT")
    return Jacobians(d, (JT,))


# ----------------------------------------------------------------- scan
LEAF_IMPL = {"auto": 0, "ffma": 1, "tensor": 2, "tensor_tf32": 3, "int8": 4}


def _opts(mode="blocked", block0=0, block=0, trace=None, leaf_impl="auto", levels=(0, 0)) -> _Opts:
    o = _Opts(MODES[mode] if isinstance(mode, str) else int(mode), int(block0), int(block),
              LEAF_IMPL[leaf_impl] if isinstance(leaf_impl, str) else int(leaf_impl))
    o.up_levels, o.down_levels = int(levels[0]), int(levels[1])
    if trace is not None:
        o.events, o.n_events, o.launches = trace._arr, len(trace.events), C.pointer(trace._count)
    return o


class LaunchTrace:
    """Per-launch CUDA events for bppsa_scan_opts.events (instrumentation):
    events[2k] / events[2k+1] bracket the library's k-th kernel launch."""

    def __init__(self, max_launches: int = 64):
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(2 * max_launches)]
        for e in self.events:          # materialise the cudaEvent_t handles
            e.record()
        torch.cuda.synchronize()
        self._arr = (_vp * len(self.events))(*[e.cuda_event for e in self.events])
        self._count = _i(0)

    @property
    def launches(self) -> int:
        return self._count.value

    def kernel_ms(self, k: int) -> float:
        return self.events[2 * k].elapsed_time(self.events[2 * k + 1])


def scan_workspace_size(jac: Jacobians, mode="blocked", block0=0, block=0, levels=(0, 0)) -> int:
    n = _sz()
    o = _opts(mode, block0, block, levels=levels)
    _check(_lib.bppsa_scan_workspace_size(C.byref(jac.desc), C.byref(o), C.byref(n)), "bppsa_scan_workspace_size")
    return n.value


def workspace(nbytes: int, device=None) -> torch.Tensor:
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device or "cuda")


def scan(jac: Jacobians, seed: torch.Tensor, grad_h: torch.Tensor | None = None,
         grad_h_init: torch.Tensor | bool | None = None, ws: torch.Tensor | None = None,
         mode="blocked", block0: int = 0, block: int = 0, stream=None, trace: LaunchTrace | None = None,
         leaf_impl="auto", levels=(0, 0)):
    """bppsa_scan: all grad_h[t] = dl/dh_t at once (and dl/dh_init if asked).
    `levels` = (up_levels, down_levels) for mode="hybrid"."""
    T, B, H = jac.T, jac.B, jac.H
    dev = seed.device
    _req(seed, (B, H), "seed")
    if grad_h is None:
        grad_h = torch.empty((T, B, H), dtype=torch.float32, device=dev)
    if grad_h_init is True:
        grad_h_init = torch.empty((B, H), dtype=torch.float32, device=dev)
    elif grad_h_init is False:
        grad_h_init = None
    _req(grad_h, (T, B, H), "grad_h", dev)
    _req(grad_h_init, (B, H), "grad_h_init", dev)
    o = _opts(mode, block0, block, trace, leaf_impl, levels)
    if ws is None:
        ws = workspace(scan_workspace_size(jac, mode, block0, block, levels), dev)
    _ws(ws, dev)
    _check(_lib.bppsa_scan(C.byref(jac.desc), _ptr(seed, "seed"), _ptr(grad_h, "grad_h"),
                           _ptr(grad_h_init, "grad_h_init"), ws.data_ptr(), ws.numel(), C.byref(o),
                           _stream(stream)), "bppsa_scan")
    return grad_h, grad_h_init


def exchange_publish(aggregate: torch.Tensor, rank: int, world: int, peer_mailboxes: torch.Tensor,
                     peer_flags: torch.Tensor, counter: torch.Tensor, acks: torch.Tensor, epoch: int, stream=None):
    """bppsa_exchange_publish: (after the readers' acks of epoch - 2) aggregate
    -> every rank's mailbox, then the flags (peer_mailboxes / peer_flags:
    int64 device arrays of device pointers; acks: this rank's ack words)."""
    _check(_lib.bppsa_exchange_publish(_ptr(aggregate, "aggregate"), aggregate.numel(), rank, world,
                                       peer_mailboxes.data_ptr(), peer_flags.data_ptr(), counter.data_ptr(),
                                       acks.data_ptr(), epoch, _stream(stream)), "bppsa_exchange_publish")


def exchange_ack(rank: int, world: int, peer_acks: torch.Tensor, epoch: int, stream=None):
    """bppsa_exchange_ack: this rank finished reading epoch `epoch`."""
    _check(_lib.bppsa_exchange_ack(rank, world, peer_acks.data_ptr(), epoch, _stream(stream)), "bppsa_exchange_ack")


def exchange_wait(flags: torch.Tensor, rank: int, world: int, epoch: int, stream=None):
    _check(_lib.bppsa_exchange_wait(flags.data_ptr(), rank, world, epoch, _stream(stream)), "bppsa_exchange_wait")


def gru_gates(x: torch.Tensor, h: torch.Tensor, W_ih3: torch.Tensor, W_hh3: torch.Tensor, b_ih3: torch.Tensor,
              b_hh3: torch.Tensor, h_init: torch.Tensor | None = None, out=None, stream=None) -> dict:
    """bppsa_gru_gates (FO): the GRU tape {h_prev, r, z, n, M} recomputed from x and h."""
    T, B, I = x.shape
    H = h.shape[2]
    _req(h, (T, B, H), "h", x.device)
    _req(W_ih3, (3 * H, I), "W_ih3", x.device)
    _req(W_hh3, (3 * H, H), "W_hh3", x.device)
    _req(b_ih3, (3 * H,), "b_ih3", x.device)
    _req(b_hh3, (3 * H,), "b_hh3", x.device)
    _req(h_init, (B, H), "h_init", x.device)
    if out is None:
        out = {k: torch.empty((T, B, H), dtype=torch.float32, device=h.device) for k in ("h_prev", "r", "z", "n", "M")}
    for k in ("h_prev", "r", "z", "n", "M"):
        _req(out[k], (T, B, H), k, x.device)
    _check(_lib.bppsa_gru_gates(T, B, H, I, _ptr(x, "x"), _ptr(h, "h"), _ptr(h_init, "h_init"), _ptr(W_ih3, "W_ih3"),
                                _ptr(W_hh3, "W_hh3"), _ptr(b_ih3, "b_ih3"), _ptr(b_hh3, "b_hh3"),
                                *[_ptr(out[k], k) for k in ("h_prev", "r", "z", "n", "M")], _stream(stream)),
           "bppsa_gru_gates")
    return out


def scan_affine(jac: Jacobians, seed: torch.Tensor, e: torch.Tensor, grad_h: torch.Tensor | None = None,
                grad_h_init: torch.Tensor | bool | None = None, ws: torch.Tensor | None = None,
                mode="blocked", block0: int = 0, block: int = 0, stream=None, trace: LaunchTrace | None = None,
                leaf_impl="auto"):
    """bppsa_scan_affine: per-step losses, e [T,B,H] = dl_t/dh_t (partial)."""
    T, B, H = jac.T, jac.B, jac.H
    dev = seed.device
    _req(seed, (B, H), "seed")
    _req(e, (T, B, H), "e", dev)
    if grad_h is None:
        grad_h = torch.empty((T, B, H), dtype=torch.float32, device=dev)
    if grad_h_init is True:
        grad_h_init = torch.empty((B, H), dtype=torch.float32, device=dev)
    elif grad_h_init is False:
        grad_h_init = None
    _req(grad_h, (T, B, H), "grad_h", dev)
    _req(grad_h_init, (B, H), "grad_h_init", dev)
    o = _opts(mode, block0, block, trace, leaf_impl)
    if ws is None:
        ws = workspace(scan_workspace_size(jac, mode, block0, block), dev)
    _ws(ws, dev)
    _check(_lib.bppsa_scan_affine(C.byref(jac.desc), _ptr(seed, "seed"), _ptr(e, "e"), _ptr(grad_h, "grad_h"),
                                  _ptr(grad_h_init, "grad_h_init"), ws.data_ptr(), ws.numel(), C.byref(o),
                                  _stream(stream)), "bppsa_scan_affine")
    return grad_h, grad_h_init


def scan_shard_up(jac: Jacobians, seed: torch.Tensor | None, aggregate: torch.Tensor, ws: torch.Tensor,
                  block0: int = 0, block: int = 0, stream=None, trace: LaunchTrace | None = None,
                  leaf_impl="auto"):
    dev = aggregate.device
    _req(seed, (jac.B, jac.H), "seed", dev)
    if aggregate.numel() != jac.B * jac.H * jac.H:
        raise ValueError(f"aggregate must hold B*H*H = {jac.B * jac.H * jac.H} floats")
    _ws(ws, dev)
    o = _opts("blocked", block0, block, trace, leaf_impl)
    _check(_lib.bppsa_scan_shard_up(C.byref(jac.desc), _ptr(seed, "seed"), _ptr(aggregate, "aggregate"),
                                    ws.data_ptr(), ws.numel(), C.byref(o), _stream(stream)), "bppsa_scan_shard_up")
    return aggregate


def scan_shard_up_publish(jac: Jacobians, seed: torch.Tensor | None, aggregate: torch.Tensor, ws: torch.Tensor,
                          rank: int, world: int, peer_mailboxes: torch.Tensor, peer_flags: torch.Tensor,
                          counter: torch.Tensor, acks: torch.Tensor, epoch: int, block0: int = 0, block: int = 0,
                          stream=None, trace: LaunchTrace | None = None, leaf_impl="auto"):
    """bppsa_scan_shard_up_publish: the shard up-sweep with the peer-memory
    publish fused into its top level (arguments of exchange_publish)."""
    dev = aggregate.device
    _req(seed, (jac.B, jac.H), "seed", dev)
    if aggregate.numel() != jac.B * jac.H * jac.H:
        raise ValueError(f"aggregate must hold B*H*H = {jac.B * jac.H * jac.H} floats")
    _ws(ws, dev)
    o = _opts("blocked", block0, block, trace, leaf_impl)
    _check(_lib.bppsa_scan_shard_up_publish(C.byref(jac.desc), _ptr(seed, "seed"), _ptr(aggregate, "aggregate"),
                                            ws.data_ptr(), ws.numel(), C.byref(o), rank, world,
                                            peer_mailboxes.data_ptr(), peer_flags.data_ptr(), counter.data_ptr(),
                                            acks.data_ptr(), epoch, _stream(stream)), "bppsa_scan_shard_up_publish")
    return aggregate


def scan_shard_down(jac: Jacobians, seed: torch.Tensor | None, gathered: torch.Tensor | None, rank: int,
                    world: int, grad_h: torch.Tensor, grad_h_init: torch.Tensor | None, ws: torch.Tensor,
                    block0: int = 0, block: int = 0, stream=None, trace: LaunchTrace | None = None):
    dev = grad_h.device
    T, B, H = jac.T, jac.B, jac.H
    _req(seed, (B, H), "seed", dev)
    if gathered is not None and gathered.numel() != world * B * H * H:
        raise ValueError(f"gathered must hold world*B*H*H = {world * B * H * H} floats")
    _req(grad_h, (T, B, H), "grad_h", dev)
    _req(grad_h_init, (B, H), "grad_h_init", dev)
    _ws(ws, dev)
    o = _opts("blocked", block0, block, trace)
    _check(_lib.bppsa_scan_shard_down(C.byref(jac.desc), _ptr(seed, "seed"), _ptr(gathered, "gathered"), rank,
                                      world, _ptr(grad_h, "grad_h"), _ptr(grad_h_init, "grad_h_init"),
                                      ws.data_ptr(), ws.numel(), C.byref(o), _stream(stream)),
           "bppsa_scan_shard_down")
    return grad_h, grad_h_init


# ----------------------------------------------------------------- weight grads
def weight_grads_workspace_size(T, B, H, I) -> int:
    n = _sz()
    _check(_lib.bppsa_weight_grads_workspace_size(T, B, H, I, C.byref(n)), "bppsa_weight_grads_workspace_size")
    return n.value


def weight_grads_rnn(x, h, grad_h, h_init=None, ws=None, out=None, stream=None):
    """bppsa_weight_grads_rnn -> (dW_ih [H,I], dW_hh [H,H], db [H])."""
    T, B, H = h.shape
    I = x.shape[2]
    dev = h.device
    _req(x, (T, B, I), "x", dev)
    _req(grad_h, (T, B, H), "grad_h", dev)
    _req(h_init, (B, H), "h_init", dev)
    if out is None:
        out = (torch.empty((H, I), device=dev), torch.empty((H, H), device=dev), torch.empty((H,), device=dev))
    if ws is None:
        ws = workspace(weight_grads_workspace_size(T, B, H, I), dev)
    _ws(ws, dev)
    dW_ih, dW_hh, db = out
    _req(dW_ih, (H, I), "dW_ih", dev)
    _req(dW_hh, (H, H), "dW_hh", dev)
    _req(db, (H,), "db", dev)
    _check(_lib.bppsa_weight_grads_rnn(T, B, H, I, _ptr(x, "x"), _ptr(h, "h"), _ptr(h_init, "h_init"),
                                       _ptr(grad_h, "grad_h"), _ptr(dW_ih, "dW_ih"), _ptr(dW_hh, "dW_hh"),
                                       _ptr(db, "db"), ws.data_ptr(), ws.numel(), _stream(stream)),
           "bppsa_weight_grads_rnn")
    return dW_ih, dW_hh, db


def weight_grads_rnn_part_rows(T, B, H, I) -> int:
    """Row granularity of bppsa_weight_grads_rnn_rows (0: not available)."""
    n = C.c_longlong()
    _check(_lib.bppsa_weight_grads_rnn_part_rows(T, B, H, I, C.byref(n)), "bppsa_weight_grads_rnn_part_rows")
    return n.value


def weight_grads_rnn_rows(x, h, grad_h, row0: int, row1: int, ws: torch.Tensor, h_init=None, stream=None):
    """bppsa_weight_grads_rnn_rows: partial slabs of rows [row0, row1) into ws."""
    T, B, H = h.shape
    I = x.shape[2]
    _req(x, (T, B, I), "x", h.device)
    _req(grad_h, (T, B, H), "grad_h", h.device)
    _req(h_init, (B, H), "h_init", h.device)
    _ws(ws, h.device)
    _check(_lib.bppsa_weight_grads_rnn_rows(T, B, H, I, _ptr(x, "x") if I else None, _ptr(h, "h"),
                                            _ptr(h_init, "h_init"), _ptr(grad_h, "grad_h"), row0, row1,
                                            ws.data_ptr(), ws.numel(), _stream(stream)),
           "bppsa_weight_grads_rnn_rows")


def weight_grads_rnn_reduce(T, B, H, I, ws: torch.Tensor, out=None, device=None, stream=None):
    """bppsa_weight_grads_rnn_reduce -> (dW_ih [H,I], dW_hh [H,H], db [H])."""
    dev = device or ws.device
    if out is None:
        out = (torch.empty((H, I), device=dev), torch.empty((H, H), device=dev), torch.empty((H,), device=dev))
    _req(out[0], (H, I), "dW_ih", ws.device)
    _req(out[1], (H, H), "dW_hh", ws.device)
    _req(out[2], (H,), "db", ws.device)
    _ws(ws, ws.device)
    _check(_lib.bppsa_weight_grads_rnn_reduce(T, B, H, I, _ptr(out[0], "dW_ih") if I else None,
                                              _ptr(out[1], "dW_hh"), _ptr(out[2], "db"), ws.data_ptr(), ws.numel(),
                                              _stream(stream)), "bppsa_weight_grads_rnn_reduce")
    return out


def weight_grads_gru(x, tape: dict, grad_h, ws=None, out=None, stream=None):
    """bppsa_weight_grads_gru -> (dW_ih3 [3H,I], dW_hh3 [3H,H], db_ih3 [3H], db_hh3 [3H])."""
    T, B, H = tape["r"].shape
    I = x.shape[2]
    dev = grad_h.device
    _req(x, (T, B, I), "x", dev)
    _req(grad_h, (T, B, H), "grad_h", dev)
    for k in ("h_prev", "r", "z", "n", "M"):
        _req(tape[k], (T, B, H), k, dev)
    if out is None:
        out = (torch.empty((3 * H, I), device=dev), torch.empty((3 * H, H), device=dev),
               torch.empty((3 * H,), device=dev), torch.empty((3 * H,), device=dev))
    if ws is None:
        ws = workspace(weight_grads_workspace_size(T, B, H, I), dev)
    _ws(ws, dev)
    a, b_, c, d = out
    for t_, shp, nm in ((a, (3 * H, I), "dW_ih3"), (b_, (3 * H, H), "dW_hh3"), (c, (3 * H,), "db_ih3"),
                        (d, (3 * H,), "db_hh3")):
        _req(t_, shp, nm, dev)
    _check(_lib.bppsa_weight_grads_gru(T, B, H, I, _ptr(x, "x"), _ptr(tape["h_prev"], "h_prev"),
                                       _ptr(tape["r"], "r"), _ptr(tape["z"], "z"), _ptr(tape["n"], "n"),
                                       _ptr(tape["M"], "M"), _ptr(grad_h, "grad_h"), _ptr(a, "dW_ih3"),
                                       _ptr(b_, "dW_hh3"), _ptr(c, "db_ih3"), _ptr(d, "db_hh3"), ws.data_ptr(),
                                       ws.numel(), _stream(stream)), "bppsa_weight_grads_gru")
    return out


# ----------------------------------------------------------------- CSR variant
class CsrPlan:
    """bppsa_csr_plan (library-owned; destroyed with this object)."""

    def __init__(self, handle, n, dims):
        self.h, self.n, self.dims = handle, n, dims      # dims[k] = dim x_k, k = 0..n

    def __del__(self):
        if getattr(self, "h", None):
            _lib.bppsa_csr_plan_destroy(self.h)
            self.h = None

    def info(self):
        c, s, k = C.c_longlong(), C.c_longlong(), _i()
        _check(_lib.bppsa_csr_plan_info(self.h, C.byref(c), C.byref(s), C.byref(k)), "bppsa_csr_plan_info")
        return {"contributions": c.value, "spmv_nnz": s.value, "kernels": k.value}

    def workspace_size(self, B, batched):
        arr = (_i * self.n)(*[int(b) for b in batched])
        n = _sz()
        _check(_lib.bppsa_csr_plan_workspace_size(self.h, B, arr, C.byref(n)), "bppsa_csr_plan_workspace_size")
        return n.value


def csr_plan_steps(plan: "CsrPlan"):
    """bppsa_csr_plan_steps: the per-step static FLOP analysis (fig:prune_symbolic)
    as a list of dicts (kind, phase, level, critical, flops, dense_flops)."""
    n = _i()
    _check(_lib.bppsa_csr_plan_steps(plan.h, None, 0, C.byref(n)), "bppsa_csr_plan_steps")
    arr = (_CsrStep * max(n.value, 1))()
    _check(_lib.bppsa_csr_plan_steps(plan.h, arr, n.value, C.byref(n)), "bppsa_csr_plan_steps")
    return [dict(kind=STEP_KIND[a.kind], phase=STEP_PHASE[a.phase], level=a.level, critical=bool(a.critical),
                 flops=a.flops, dense_flops=a.dense_flops) for a in arr[:n.value]]


def csr_conv3x3_build_size(ci, co, h, w, drop_zero=False):
    """-> (max_nnz, workspace bytes) of bppsa_csr_conv3x3_build (host call)."""
    nnz, ws = C.c_longlong(), _sz()
    _check(_lib.bppsa_csr_conv3x3_build_size(ci, co, h, w, int(drop_zero), C.byref(nnz), C.byref(ws)),
           "bppsa_csr_conv3x3_build_size")
    return nnz.value, ws.value


def csr_conv3x3_build(ci, co, h, w, weights: torch.Tensor | None = None, drop_zero=False, with_data=False,
                      ws=None, stream=None):
    """Device analytical conv J^T builder -> (indptr [ci h w + 1] int64, indices int32,
    tap int32, data fp32 or None), trimmed to the nnz (one host read of indptr[-1]
    when drop_zero)."""
    dev = weights.device if weights is not None else torch.device("cuda")
    cap, wsb = csr_conv3x3_build_size(ci, co, h, w, drop_zero)
    ip = torch.empty(ci * h * w + 1, dtype=torch.int64, device=dev)
    ix = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    tap = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    data = torch.empty(max(cap, 1), dtype=torch.float32, device=dev) if with_data else None
    if ws is None:
        ws = workspace(wsb, dev)
    _check(_lib.bppsa_csr_conv3x3_build(ci, co, h, w, _ptr(weights, "weights"), int(drop_zero), ip.data_ptr(),
                                        ix.data_ptr(), tap.data_ptr(), _ptr(data, "data"), ws.data_ptr(),
                                        ws.numel(), _stream(stream)), "bppsa_csr_conv3x3_build")
    nnz = int(ip[-1]) if drop_zero else cap
    return ip, ix[:nnz], tap[:nnz], None if data is None else data[:nnz]


def csr_maxpool_build(c, h, w, device=None, stream=None):
    dev = device or torch.device("cuda")
    ip = torch.empty(c * h * w + 1, dtype=torch.int64, device=dev)
    ix = torch.empty(c * h * w, dtype=torch.int32, device=dev)
    _check(_lib.bppsa_csr_maxpool_build(c, h, w, ip.data_ptr(), ix.data_ptr(), _stream(stream)),
           "bppsa_csr_maxpool_build")
    return ip, ix


def csr_identity_build(d, device=None, stream=None):
    dev = device or torch.device("cuda")
    ip = torch.empty(d + 1, dtype=torch.int64, device=dev)
    ix = torch.empty(d, dtype=torch.int32, device=dev)
    _check(_lib.bppsa_csr_identity_build(d, ip.data_ptr(), ix.data_ptr(), _stream(stream)),
           "bppsa_csr_identity_build")
    return ip, ix


def _csr_pattern_array(patterns):
    import numpy as np
    n = len(patterns)
    keep = []
    arr = (_CsrPat * n)()
    for k, (rows, cols, ip, ix) in enumerate(patterns):
        ip = np.ascontiguousarray(ip, dtype=np.int64)
        ix = np.ascontiguousarray(ix, dtype=np.int32)
        keep += [ip, ix]
        arr[k] = _CsrPat(rows, cols, int(ip[-1]), ip.ctypes.data, ix.ctypes.data)
    return arr, keep


def csr_plan_create(patterns, up_levels: int, down_levels: int, max_contributions: int = 0) -> CsrPlan:
    """patterns: [(rows, cols, indptr int64 ndarray, indices int32 ndarray)] for
    J_1^T .. J_n^T (time order)."""
    arr, keep = _csr_pattern_array(patterns)
    h = _vp()
    _check(_lib.bppsa_csr_plan_create(arr, len(patterns), up_levels, down_levels, max_contributions, C.byref(h)),
           "bppsa_csr_plan_create")
    dims = [patterns[0][0]] + [p[1] for p in patterns]
    return CsrPlan(h, len(patterns), dims)


def csr_plan_create_symbolic(patterns, up_levels: int, down_levels: int) -> CsrPlan:
    """bppsa_csr_plan_create_symbolic: the schedule's static analysis only
    (info / steps; host-only, no device memory), for schedules whose
    contribution lists do not fit."""
    arr, keep = _csr_pattern_array(patterns)
    h = _vp()
    _check(_lib.bppsa_csr_plan_create_symbolic(arr, len(patterns), up_levels, down_levels, C.byref(h)),
           "bppsa_csr_plan_create_symbolic")
    dims = [patterns[0][0]] + [p[1] for p in patterns]
    return CsrPlan(h, len(patterns), dims)


def csr_scan(plan: CsrPlan, data, batched, seed, grads=None, ws=None, stream=None):
    """bppsa_csr_scan.  data[k]: device values of J_{k+1}^T ([nnz] shared or
    [nnz, B] sample-minor); seed [B, dim x_n].  Returns grads[k] = dl/dx_k
    ([B, dim x_k], k = 0..n)."""
    B = seed.shape[0]
    if grads is None:
        grads = [torch.empty((B, d), dtype=torch.float32, device=seed.device) for d in plan.dims]
    if ws is None:
        ws = workspace(plan.workspace_size(B, batched), seed.device)
    darr = (_vp * plan.n)(*[_ptr(d, f"data[{k}]") for k, d in enumerate(data)])
    garr = (_vp * (plan.n + 1))(*[None if g is None else _ptr(g, "grad") for g in grads])
    barr = (_i * plan.n)(*[int(b) for b in batched])
    _check(_lib.bppsa_csr_scan(plan.h, B, darr, barr, _ptr(seed, "seed"), garr, ws.data_ptr(), ws.numel(),
                               _stream(stream)), "bppsa_csr_scan")
    return grads


def csr_conv3x3_pattern(ci, co, h, w, weights=None, drop_zero=False):
    """Host pattern of a 3x3/pad-1 conv J^T -> (indptr int64, indices int32, tap int32)."""
    import numpy as np
    wt = None if weights is None else np.ascontiguousarray(weights, dtype=np.float32)
    wp = None if wt is None else wt.ctypes.data
    nnz = C.c_longlong()
    _check(_lib.bppsa_csr_conv3x3_pattern(ci, co, h, w, wp, int(drop_zero), C.byref(nnz), None, None, None),
           "bppsa_csr_conv3x3_pattern")
    ip = np.empty(ci * h * w + 1, np.int64)
    ix = np.empty(nnz.value, np.int32)
    tap = np.empty(nnz.value, np.int32)
    _check(_lib.bppsa_csr_conv3x3_pattern(ci, co, h, w, wp, int(drop_zero), C.byref(nnz), ip.ctypes.data,
                                          ix.ctypes.data, tap.ctypes.data), "bppsa_csr_conv3x3_pattern")
    return ip, ix, tap


def csr_conv_data(tap: torch.Tensor, weights: torch.Tensor, out=None, stream=None):
    if out is None:
        out = torch.empty(tap.numel(), dtype=torch.float32, device=tap.device)
    _check(_lib.bppsa_csr_conv_data(tap.numel(), tap.data_ptr(), _ptr(weights, "weights"), _ptr(out, "data"),
                                    _stream(stream)), "bppsa_csr_conv_data")
    return out


def csr_relu_data(x: torch.Tensor, out=None, stream=None):
    """x [B, d] (ReLU inputs) -> data [d, B] in {0, 1} (Alg. 7)."""
    B, d = x.shape[0], x[0].numel()
    if out is None:
        out = torch.empty((d, B), dtype=torch.float32, device=x.device)
    _check(_lib.bppsa_csr_relu_data(d, B, _ptr(x, "x"), _ptr(out, "data"), _stream(stream)), "bppsa_csr_relu_data")
    return out


def csr_maxpool_pattern(c, h, w):
    import numpy as np
    ip = np.empty(c * h * w + 1, np.int64)
    ix = np.empty(c * h * w, np.int32)
    _check(_lib.bppsa_csr_maxpool_pattern(c, h, w, ip.ctypes.data, ix.ctypes.data), "bppsa_csr_maxpool_pattern")
    return ip, ix


def csr_maxpool_data(pool_idx: torch.Tensor, c, h, w, out=None, stream=None):
    """pool_idx [B, c, h/2, w/2] int64 (torch return_indices) -> data [c*h*w, B]."""
    B = pool_idx.shape[0]
    if out is None:
        out = torch.empty((c * h * w, B), dtype=torch.float32, device=pool_idx.device)
    assert pool_idx.dtype == torch.int64 and pool_idx.is_contiguous()
    _check(_lib.bppsa_csr_maxpool_data(c, h, w, B, pool_idx.data_ptr(), _ptr(out, "data"), _stream(stream)),
           "bppsa_csr_maxpool_data")
    return out
