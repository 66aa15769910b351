#!/usr/bin/env python
"""bench.py — BPPSA backward (arXiv 1907.10134) on B200.

Metric (BASELINE.json): BPPSA backward ms vs sequential BP (1/2/4/8 GPU);
% HBM/tensor roofline.  One "step" = one full backward pass of the hot path
over one batch: fused RNN leaves (a1) + blocked Blelloch up-sweep (a2) + root
reset (a3) + down-sweep (a4) + carry exchange (a5, N > 1) + weight gradients
(a6).  Default workload = config 4 (tanh RNN, H = 64, B = 16, T = 2^20), the
configuration BASELINE.json shards across 1/2/4/8 B200s (strong scaling: the
total sequence is fixed, rank r owns T/N contiguous steps).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--quick]

Rank 0 prints ONE JSON line.  With --gpus N > 1 and no torchrun environment
the script relaunches itself as N ranks (torch.distributed.run, 127.0.0.1).
`--impl reference` times the fp64 CPU oracle (oracle/, the reference arm of
this tier) on the full C4 workload once (steps = 1).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BPPSA backward ms vs sequential BP (1/2/4/8 GPU); % HBM/tensor roofline"
C4 = dict(T=1 << 20, B=16, H=64, I=1)
C4_BLOCK0, C4_BLOCK = 1024, 32
E2E_BLOCK0 = 256        # the streamed e2e path: a short last-chunk walk (DESIGN "Host inputs")


def c4_block0(world: int) -> int:
    """Level-0 block per rank for time shards of 2^20 / world steps, measured
    on one B200 (DESIGN "Multi-GPU"): the int8 walk runs one 128-chain tile per
    SM for block0 dependent steps, so its time is ~ceil(tiles / 148) x block0
    step times; the level-1 fold shrinks with fewer blocks.  Full scan of the
    shard, ring fold (scripts/block0_sweep.py, r02): N = 1: 512 44.00 / 1024
    43.67 / 2048 44.89 ms; N = 2 (T = 2^19): 256 22.27 / 512 21.88 / 1024
    22.13; N = 4: 128 11.32 / 256 10.91 / 512 11.13; N = 8: 128 5.87 / 256
    5.68 / 512 6.78."""
    return {1: 1024, 2: 512}.get(world, 256)
SMALL = {   # secondary configs (N = 1 sweep): (T, B, H, block0, block)
    "c1": dict(T=1000, B=16, H=20, block0=8, block=8),
    "c2": dict(T=30000, B=16, H=20, block0=32, block=16),   # r02g: 0.44 ms (0.48 at block0 64, 0.48 at 16; kbench)
}
FP32_LANES_PER_SM, N_SM = 128, 148


def c4_inputs(seed: int = 0):
    """C4 inputs through the host numpy forward (the parity tests' inputs)."""
    import bppsa_workloads as W
    return W.rnn_workload(C4["T"], C4["B"], C4["H"], seed=seed, I=C4["I"])


def c4_inputs_gpu(seed: int, dev):
    """C4 inputs for the bench, same recipe as bppsa_workloads.rnn_workload
    (seeded bitstreams, torch-default init, fp32 forward, mean-CE head seed)
    but with the forward on the GPU: torch nn.RNN (cuDNN, TF32 off) over
    32768-step chunks carrying the state, so every rank builds its inputs in
    well under a second instead of a 2^20-step host loop.  Returns device x,
    h (full length) and host params / seed."""
    import torch
    import bppsa_workloads as W
    T, B, H, I = C4["T"], C4["B"], C4["H"], C4["I"]
    x_np, labels = W.bitstreams(T, B, seed)
    p = W.rnn_params(H, I, 10, seed + 1)
    rnn = torch.nn.RNN(I, H, nonlinearity="tanh").to(dev)
    with torch.no_grad():
        for name, key in (("weight_ih_l0", "W_ih"), ("weight_hh_l0", "W_hh"), ("bias_ih_l0", "b_ih"),
                          ("bias_hh_l0", "b_hh")):
            getattr(rnn, name).copy_(torch.from_numpy(p[key]))
        x = torch.from_numpy(x_np).to(dev)
        h = torch.empty((T, B, H), device=dev)
        state = torch.zeros((1, B, H), device=dev)
        for t0 in range(0, T, 1 << 15):
            out, state = rnn(x[t0:t0 + (1 << 15)], state)
            h[t0:t0 + out.shape[0]] = out
    g = W.head_seed(h[-1].cpu().numpy(), p["W_out"], p["b_out"], labels)
    return x, h, p, g


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "bf16_tflops": 1590.0, "source": "fallback"}
    f = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(f):
        d = json.load(open(f))
        p.update(hbm_gbs=d.get("hbm_gbs", p["hbm_gbs"]), sm_max_mhz=d.get("sm_max_mhz", p["sm_max_mhz"]),
                 bf16_tflops=d.get("bf16_tflops", p["bf16_tflops"]), source="MEASURED_PEAKS.json")
    # FP32 FFMA pipe: 148 SMs x 128 lanes x 2 flop x f_SM
    p["fp32_tflops"] = N_SM * FP32_LANES_PER_SM * 2 * p["sm_max_mhz"] * 1e6 / 1e12
    return p


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def level0_flops(T: int, B: int, H: int, C0: int, head: bool) -> float:
    """Algorithmic flops of the level-0 fold (the dominant kernel): folding a
    block of l matrices takes l-1 GEMMs (2H^3); the head block (seed + l-1
    leaves) takes l-1 GEMVs (2H^2); building each leaf J^T = W^T diag(d) is H^2."""
    S = T + (1 if head else 0)
    nblk = -(-S // C0)
    gemm = gemv = 0
    for q in range(nblk):
        ln = min(C0, S - q * C0)
        if head and q == 0:
            gemv += ln - 1
        else:
            gemm += ln - 1
    return B * (gemm * 2.0 * H ** 3 + gemv * 2.0 * H ** 2 + T * H ** 2)


def scan_alg_counts(T: int, B: int, H: int, I: int = 1, gru: bool = False):
    """Algorithmic work of one full backward: Alg. 1's n - L
    GEMMs (2H^3) and n - 1 GEMVs (2H^2) per sample (n = T slots of leaves,
    L = ceil(log2(n + 1))), the leaves (H^2 per step RNN, 6H^2 + H GRU), the
    weight gradients 2 B T H (H + I + 1) (x3 GRU); fused bytes: activations
    read once + grad_h written once (8H per element RNN, 24H GRU) + the
    weight-gradient reads 4 B T (2H + I)."""
    n, L = T, max(1, math.ceil(math.log2(T + 1)))
    leaf = (6 * H * H + H) if gru else H * H
    scan = B * ((n - L) * 2.0 * H ** 3 + (n - 1) * 2.0 * H ** 2 + n * leaf)
    wg = (3 if gru else 1) * 2.0 * B * T * H * (H + I + 1)
    bytes_ = B * T * ((24 if gru else 8) * H) + 4.0 * B * T * (2 * H + I)
    return scan + wg, bytes_


def graph_launch_us(n: int = 64):
    """Latency floor unit: one dependent kernel node of a replayed CUDA graph
    (tiny kernels back to back on one stream), measured on this GPU."""
    import torch
    a = torch.zeros(1, device="cuda")

    def chain():
        for _ in range(n):
            a.add_(1.0)
    chain()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            chain()
    torch.cuda.synchronize()
    return _time(gr.replay, reps=20) * 1e3 / n


def roofline_small(ms: float, flops: float, bytes_: float, launches: int, launch_us: float, pk: dict):
    """ALU (FFMA pipe), HBM and latency-floor fractions of a latency-bound config."""
    return {"bound": "latency",
            "alu": {"achieved_tflops": round(flops / (ms * 1e-3) / 1e12, 3), "peak_tflops": round(pk["fp32_tflops"], 1),
                    "frac": round(flops / (ms * 1e-3) / 1e12 / pk["fp32_tflops"], 4)},
            "hbm": {"achieved_gbs": round(bytes_ / (ms * 1e-3) / 1e9, 1), "peak_gbs": pk["hbm_gbs"],
                    "frac": round(bytes_ / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], 4)},
            "latency_floor_ms": round(launches * launch_us * 1e-3, 4), "launches": launches,
            "launch_us": round(launch_us, 3),
            "frac": round(launches * launch_us * 1e-3 / ms, 4),
            "algorithmic_flops": flops, "algorithmic_bytes": bytes_}


def load_traffic(kernel: str):
    f = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(f):
        d = json.load(open(f))
        v = d.get(kernel)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch")
    return None


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1907_10134_b200 import api
    from paper_1907_10134_b200.dist import CudaShardBackend, shard_bounds, sharded_scan

    world, rank, local = dist_env()
    # dev aid: BPPSA_BENCH_DEVICE pins every rank to one GPU and
    # BPPSA_BENCH_BACKEND=gloo lets several ranks share it (NCCL refuses) —
    # how the N > 1 path is exercised on a one-GPU box; the driver's runs use
    # one GPU per rank over NCCL (the defaults)
    if os.environ.get("BPPSA_BENCH_DEVICE") is not None:
        local = int(os.environ["BPPSA_BENCH_DEVICE"])
    backend = os.environ.get("BPPSA_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    if world > 1:
        if backend == "nccl":
            # the communicator-init lines on stderr let the driver count the ranks
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    T, B, H, I = C4["T"], C4["B"], C4["H"], C4["I"]
    lo, hi = shard_bounds(T, world)[rank]
    head = rank == world - 1
    dev = torch.device("cuda", local)
    x_full, h_full, params, g_np = c4_inputs_gpu(args.seed, dev)
    h = h_full[lo:hi].clone()                 # this rank's shard only
    x = x_full[lo:hi].clone()
    h_init = h_full[lo - 1].clone() if lo > 0 else None
    Whh = torch.from_numpy(params["W_hh"]).to(dev)
    g = torch.from_numpy(g_np).to(dev) if head else None
    host = None
    if world == 1 and not args.quick:         # e2e / sequential baselines need host copies
        host = dict(h=h_full.cpu().numpy(), x=x_full.cpu().numpy(), W_hh=params["W_hh"], g=g_np)
    del x_full, h_full
    torch.cuda.empty_cache()
    Tl = hi - lo
    jac = api.jacobians_rnn(h, Whh)
    grad = torch.empty((Tl, B, H), device=dev)
    wout = (torch.empty((H, I), device=dev), torch.empty((H, H), device=dev), torch.empty((H,), device=dev))
    ws_w = api.workspace(api.weight_grads_workspace_size(Tl, B, H, I), dev)
    b0 = c4_block0(world)
    backend = CudaShardBackend(jac, b0, C4_BLOCK) if world > 1 else None
    # carry exchange: NCCL all-gather (default) or BPPSA_EXCHANGE=peer, the
    # peer-memory mailboxes of bppsa_exchange_publish / _wait
    exchange = None
    if world > 1 and os.environ.get("BPPSA_EXCHANGE", "nccl") == "peer":
        from paper_1907_10134_b200.dist import PeerExchange
        exchange = PeerExchange(B, H)
    ws = api.workspace(api.scan_workspace_size(jac, "blocked", b0, C4_BLOCK), dev) if world == 1 else None

    def step(trace=None):
        if world == 1:
            api.scan(jac, g, grad_h=grad, ws=ws, block0=b0, block=C4_BLOCK, trace=trace)
        else:
            sharded_scan(_Traced(backend, trace), g, grad_h=grad, exchange=exchange)
        dWih, dWhh, db = api.weight_grads_rnn(x, h, grad, h_init=h_init, ws=ws_w, out=wout)
        if world > 1:
            for t_ in (dWih, dWhh, db):
                dist.all_reduce(t_)
        return dWih, dWhh, db

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    traces = [api.LaunchTrace(32) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for k in range(args.steps):
            step(traces[k])
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    # dominant kernel: launch 0 (level-0 fused leaf fold) of every step
    k0 = [t.kernel_ms(0) for t in traces]
    kall = [[t.kernel_ms(i) for i in range(t.launches)] for t in traces]
    launches_scan = traces[0].launches
    if world > 1:
        tt = torch.tensor([ms, statistics.mean(k0)], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, k0m = float(tt[0]), float(tt[1])
    else:
        k0m = statistics.mean(k0)
    result = dict(ms=ms, k0_ms=k0m, kernels_ms=[statistics.mean(col) for col in zip(*kall)],
                  launches=launches_scan + 2, clocks=clk.summary(), Tl=Tl, head=head)
    if rank == 0:
        pk = peaks()
        flops = level0_flops(Tl, B, H, b0, head)
        achieved = flops / (k0m * 1e-3) / 1e12
        # the level-0 fold runs on tcgen05 kind::i8 with exact s32 accumulation:
        # x as 3 and W as 4 8-bit digits, the digit products with i + j <= 3 =
        # 9 int8 MACs per fp32 MAC (tc_i8.cu); int8 dense peak = 2 x the
        # measured bf16 peak (B200_PROFILING.md: fp8/int8 4.5 vs bf16 2.25 PF
        # nominal), so the fp32-faithful peak of this kernel is that / 9
        i8_peak = 2.0 * pk["bf16_tflops"]
        peak = i8_peak / 9.0
        result["roofline"] = {"bound": "tensor",
                              "kernel": "tc_fold_i8r_kernel (level-0 fused fold, tcgen05 kind::i8, exact s32 "
                                        "accumulation of 8-bit digit products; 4 tiles over 2 TMEM accumulators)",
                              "achieved": round(achieved, 3), "peak": round(peak, 2),
                              "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                              # the ncu capture is of the single-GPU launch (T = 2^20)
                              "traffic": load_traffic("tc_fold_i8") if world == 1 else None,
                              "algorithmic_flops_per_launch": flops,
                              "peak_note": "fp32-faithful int8-digit peak = 2 x measured bf16 dense %.1f TF (%s) "
                                           "= %.1f int8 TOPS / 9 digit products per fp32 MAC; for comparison the "
                                           "FFMA-pipe peak %.1f TF (exact fp32 on CUDA cores) and the biased "
                                           "3xFP16 peak %.1f TF" % (pk["bf16_tflops"], pk["source"], i8_peak,
                                                                   pk["fp32_tflops"], pk["bf16_tflops"] / 3.0),
                              "share_of_step": round(k0m / ms, 4)}
    if world == 1 and not args.quick:
        result["e2e"] = e2e_ours(api, host, args)
        result["sequential_bp"] = sequential_baselines(api, host, args)
        result["sweep"] = sweep_small(api, args)
        # NEXT-4: the affine scan (a loss on every step) on the same C4 inputs
        gen = torch.Generator(device=dev).manual_seed(args.seed)
        e_steps = torch.randn((T, B, H), device=dev, generator=gen) * 0.01
        aff = _time(lambda: api.scan_affine(jac, g, e_steps, grad_h=grad, ws=ws, block0=b0,
                                            block=C4_BLOCK), reps=5, warm=2)
        plain = _time(lambda: api.scan(jac, g, grad_h=grad, ws=ws, block0=b0, block=C4_BLOCK), reps=5, warm=2)
        result["affine"] = {"workload": "C4 shapes, per-step losses e ~ 0.01 N(0,1) (synthetic)",
                            "scan_affine_ms": round(aff, 3), "scan_ms": round(plain, 3)}
        del e_steps
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


class _Traced:
    """Forward the LaunchTrace into the shard backend's library calls."""

    def __init__(self, backend, trace):
        self.b, self.trace = backend, trace

    def up(self, seed):
        import torch
        B, H = self.b.jac.B, self.b.jac.H
        agg = torch.empty((B, H * H), device="cuda")
        self.b.api.scan_shard_up(self.b.jac, seed, agg, self.b.ws, self.b.block0, self.b.block, trace=self.trace)
        return agg

    def down(self, seed, gathered, rank, world, grad_h=None, want_init=False):
        self.b.api.scan_shard_down(self.b.jac, seed, gathered, rank, world, grad_h, None, self.b.ws,
                                   self.b.block0, self.b.block)
        return grad_h, None


def e2e_ours(api, w, args):
    """Same backward through the public API with HOST inputs: pinned H2D of the
    step's inputs (h, x, W_hh, seed) + the backward + D2H of the step's result
    (dW_ih, dW_hh, db, dl/dh_init), all inside the timed region.  The copy of h
    (4.3 GB) is the long pole, so the backward runs on time chunks as they land
    (paper_1907_10134_b200/stream.py: chunked shard up/down sweeps in reverse
    time order on a second stream)."""
    import torch
    from paper_1907_10134_b200.stream import StreamedRnnBackward
    T, B, H, I = C4["T"], C4["B"], C4["H"], C4["I"]
    hp = torch.from_numpy(w["h"]).pin_memory()
    xp = torch.from_numpy(w["x"]).pin_memory()
    Wp = torch.from_numpy(w["W_hh"]).pin_memory()
    gp = torch.from_numpy(w["g"]).pin_memory()
    outs_h = [torch.empty(s, pin_memory=True) for s in ((H, I), (H, H), (H,), (B, H))]
    chunks = 16
    sb = StreamedRnnBackward(T, B, H, I, chunks=chunks, block0=E2E_BLOCK0, block=C4_BLOCK)

    def step():
        sb.run(hp, xp, Wp, gp, out_host=outs_h)

    step()
    torch.cuda.synchronize()
    n = max(1, min(args.steps, 3))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    torch.cuda.synchronize()
    h2d = sum(t.numel() * 4 for t in (hp, xp, Wp, gp))
    d2h = sum(t.numel() * 4 for t in outs_h)
    res = {"value": round(e0.elapsed_time(e1) / n, 3), "unit": "ms", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": n,
           "path": f"StreamedRnnBackward ({sb.G} time chunks: pinned H2D overlapped with "
                   f"bppsa_scan_shard_up/_down and the weight-gradient rows of each chunk, then the "
                   f"fixed-order reduction)"}
    # the H2D alone, for reference: the floor of this e2e number
    hd = torch.empty_like(hp, device="cuda")
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    hd.copy_(hp, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    res["h2d_h_only_ms"] = round(c0.elapsed_time(c1), 3)
    del hd, sb
    torch.cuda.empty_cache()
    return res


def cudnn_backward_ms(T, B, H, I, reps=3, x=None, seed=0, gru=False):
    """The paper's comparator: torch nn.RNN / nn.GRU (cuDNN)
    backward through time, timed from loss.backward() start to end."""
    import torch
    torch.manual_seed(seed)
    m = (torch.nn.GRU(I, H) if gru else torch.nn.RNN(I, H, nonlinearity="tanh")).cuda()
    head = torch.nn.Linear(H, 11 if gru else 10).cuda()
    xs = torch.from_numpy(x).cuda() if x is not None else (torch.rand(T, B, I, device="cuda") < 0.5).float()
    labels = torch.randint(0, 10, (B,), device="cuda")
    times = []
    for r in range(reps + 1):
        out, _ = m(xs)
        loss = torch.nn.functional.cross_entropy(head(out[-1]), labels)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        loss.backward()
        e1.record()
        torch.cuda.synchronize()
        if r > 0:
            times.append(e0.elapsed_time(e1))
        m.zero_grad(set_to_none=True)
    return statistics.median(times)


def sequential_baselines(api, w, args):
    """Sequential BP on the same GPU: our LINEAR mode (one warp per sample walks
    all T steps: the best sequential GEMV chain) and cuDNN (extrapolated from
    T = 2^16; its backward is linear in T)."""
    import torch
    T, B, H = C4["T"], C4["B"], C4["H"]
    h = torch.from_numpy(w["h"]).cuda()
    Whh = torch.from_numpy(w["W_hh"]).cuda()
    g = torch.from_numpy(w["g"]).cuda()
    jac = api.jacobians_rnn(h, Whh)
    grad = torch.empty((T, B, H), device="cuda")
    ws = api.workspace(api.scan_workspace_size(jac, "linear"))
    api.scan(jac, g, grad_h=grad, ws=ws, mode="linear")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    api.scan(jac, g, grad_h=grad, ws=ws, mode="linear")
    e1.record()
    torch.cuda.synchronize()
    lin = e0.elapsed_time(e1)
    del h, grad, ws
    torch.cuda.empty_cache()
    cud, note = None, "cuDNN rejected every tried T"
    for Ts in (1 << 16, 1 << 15, 1 << 14, 1 << 13, 1 << 12):
        try:
            cud = cudnn_backward_ms(Ts, B, H, 1, reps=2) * (T / Ts)
            note = f"torch nn.RNN backward (cuDNN, TF32 off) at T={Ts}, x{T // Ts} (linear in T)"
            break
        except RuntimeError as ex:  # cuDNN refuses very long sequences
            note = f"T={Ts}: {str(ex)[:80]}"
            torch.cuda.empty_cache()
    return {"gpu_linear_scan_ms": round(lin, 3), "cudnn_backward_ms": None if cud is None else round(cud, 3),
            "cudnn_note": note,
            "gpu_linear_note": "bppsa_scan mode=LINEAR: sequential BP, one warp per sample, scan only"}


def _time(fn, reps=20, warm=3):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def sweep_small(api, args):
    """Configs 1-3 on one GPU: BPPSA full backward (scan + weight grads),
    CUDA-graph replayed; our GPU linear scan; cuDNN backward."""
    import torch
    import bppsa_workloads as W
    out = {}
    pk = peaks()
    launch_us = graph_launch_us()
    out["graph_node_us"] = round(launch_us, 3)
    for name, c in SMALL.items():
        w = W.rnn_workload(c["T"], c["B"], c["H"], seed=1)
        h, x = torch.from_numpy(w.h).cuda(), torch.from_numpy(w.x).cuda()
        Whh, g = torch.from_numpy(w.W_hh).cuda(), torch.from_numpy(w.g).cuda()
        jac = api.jacobians_rnn(h, Whh)
        grad = torch.empty_like(h)
        ws = api.workspace(api.scan_workspace_size(jac, "blocked", c["block0"], c["block"]))
        wsl = api.workspace(api.scan_workspace_size(jac, "linear"))
        ws_w = api.workspace(api.weight_grads_workspace_size(c["T"], c["B"], c["H"], 1))
        wout = (torch.empty((c["H"], 1), device="cuda"), torch.empty((c["H"], c["H"]), device="cuda"),
                torch.empty((c["H"],), device="cuda"))

        def bwd():
            api.scan(jac, g, grad_h=grad, ws=ws, block0=c["block0"], block=c["block"])
            api.weight_grads_rnn(x, h, grad, ws=ws_w, out=wout)

        eager = _time(bwd)
        graph_ms = None
        try:
            gr = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                bwd()
                torch.cuda.synchronize()
                with torch.cuda.graph(gr, stream=s, capture_error_mode="relaxed"):
                    bwd()
            torch.cuda.synchronize()
            graph_ms = _time(gr.replay)
        except Exception as ex:  # noqa: BLE001
            graph_ms = f"capture failed: {ex}"[:120]
        lin = _time(lambda: api.scan(jac, g, grad_h=grad, ws=wsl, mode="linear"), reps=5)
        cud = cudnn_backward_ms(c["T"], c["B"], c["H"], 1, reps=5)
        tr = api.LaunchTrace(64)
        api.scan(jac, g, grad_h=grad, ws=ws, block0=c["block0"], block=c["block"], trace=tr)
        torch.cuda.synchronize()
        nl = tr.launches + 2                      # + the weight-gradient partials and reduction
        flops, bytes_ = scan_alg_counts(c["T"], c["B"], c["H"])
        best = graph_ms if not isinstance(graph_ms, str) else eager
        out[name] = {"T": c["T"], "B": c["B"], "H": c["H"], "bppsa_ms_eager": round(eager, 4),
                     "bppsa_ms_graph": graph_ms if isinstance(graph_ms, str) else round(graph_ms, 4),
                     "gpu_linear_scan_ms": round(lin, 4), "cudnn_backward_ms": round(cud, 4),
                     "roofline": roofline_small(best, flops, bytes_, nl, launch_us, pk)}
    # config 3: GRU, H = 20, IRMAS L set (1034 x 12), B = 64
    gw = W.gru_workload("L", 64, seed=2)
    tape = {k: torch.from_numpy(v).cuda() for k, v in gw.tape.items()}
    x = torch.from_numpy(gw.x).cuda()
    W3, g = torch.from_numpy(gw.params["W_hh3"]).cuda(), torch.from_numpy(gw.g).cuda()
    jac = api.jacobians_gru(tape["h_prev"], tape["r"], tape["z"], tape["n"], tape["M"], W3)
    grad = torch.empty_like(tape["r"])
    ws = api.workspace(api.scan_workspace_size(jac, "blocked", 16, 16))
    ws_w = api.workspace(api.weight_grads_workspace_size(*grad.shape, x.shape[2]))

    def bwd_gru():
        api.scan(jac, g, grad_h=grad, ws=ws, block0=16, block=16)
        api.weight_grads_gru(x, tape, grad, ws=ws_w)

    t3 = _time(bwd_gru)
    tr = api.LaunchTrace(64)
    api.scan(jac, g, grad_h=grad, ws=ws, block0=16, block=16, trace=tr)
    torch.cuda.synchronize()
    flops, bytes_ = scan_alg_counts(1034, 64, 20, I=12, gru=True)
    out["c3"] = {"set": "L (1034 x 12)", "B": 64, "H": 20, "bppsa_ms_eager": round(t3, 4),
                 "cudnn_backward_ms": round(cudnn_backward_ms(1034, 64, 20, 12, reps=5, x=gw.x, gru=True), 4),
                 "roofline": roofline_small(t3, flops, bytes_, tr.launches + 2, launch_us, pk)}
    out["c5"] = sweep_csr(api, pk)
    out["train"] = sweep_train()
    out["hybrid"] = sweep_hybrid(api)
    out["jacgen"] = sweep_jacgen(api)
    return out


def sweep_jacgen(api, sample_cols: int = 256):
    """SURVEY 8(f) NEXT-3 / Table 1's last column: the
    analytical device builders (pattern + data of J^T, one sample) vs
    generating J^T through torch autograd one column at a time on the same
    GPU.  The autograd side is timed on `sample_cols` columns and scaled to
    all columns (one backward per output element; stated in the output)."""
    import torch
    torch.manual_seed(0)
    res = {}
    x = torch.randn(1, 3, 32, 32, device="cuda")
    conv = torch.nn.Conv2d(3, 64, 3, padding=1, bias=False).cuda()
    wflat = conv.weight.detach().reshape(-1).contiguous()
    a = torch.randn(1, 64, 32, 32, device="cuda")
    ws = api.workspace(api.csr_conv3x3_build_size(3, 64, 32, 32)[1])

    def conv_build():
        api.csr_conv3x3_build(3, 64, 32, 32, wflat, with_data=True, ws=ws)

    def relu_build():
        api.csr_identity_build(64 * 32 * 32)
        api.csr_relu_data(a.reshape(1, -1))

    _, pidx = torch.nn.functional.max_pool2d(a, 2, return_indices=True)

    def pool_build():
        api.csr_maxpool_build(64, 32, 32)
        api.csr_maxpool_data(pidx, 64, 32, 32)

    def autograd_ms(f, inp):
        inp = inp.clone().requires_grad_(True)
        y = f(inp).reshape(-1)
        cols = y.numel()
        idx = torch.randperm(cols, device="cuda")[:sample_cols].tolist()

        def run():
            for j in idx:
                torch.autograd.grad(y[j], inp, retain_graph=True)

        return _time(run, reps=2, warm=1) / len(idx) * cols, cols

    cases = {"conv1 (3->64, 32x32)": (conv_build, lambda t: conv(t), x),
             "relu1 (64x32x32)": (relu_build, torch.relu, a),
             "pool1 (64x32x32, 2x2)": (pool_build, lambda t: torch.nn.functional.max_pool2d(t, 2), a)}
    for name, (build, f, inp) in cases.items():
        an = _time(build, reps=20)
        ag, cols = autograd_ms(f, inp)
        res[name] = {"analytical_ms": round(an, 4), "autograd_column_ms_extrapolated": round(ag, 1),
                     "columns": cols, "speedup": round(ag / an, 1)}
    return {"sample_cols": sample_cols, "device": "same B200 for both", "ops": res,
            "paper_speedups_cpu_context": {"conv": 8.3e3, "relu": 1.2e6, "pool": 1.5e5}}


def sweep_hybrid(api):
    """the level-balanced hybrid on C1's
    materialised leaves (T = 1000, B = 16, H = 20): scan ms per
    (up_levels, down_levels), CUDA-graph replayed, next to the blocked
    scan on the same DENSE descriptor."""
    import torch
    import bppsa_workloads as W
    T, B, H = 1000, 16, 20
    w = W.rnn_workload(T, B, H, seed=1)
    JT = torch.empty((T, B, H, H), device="cuda")
    api.jacobians_rnn(torch.from_numpy(w.h).cuda(), torch.from_numpy(w.W_hh).cuda(), JT_out=JT)
    jac = api.jacobians_dense(JT)
    g = torch.from_numpy(w.g).cuda()
    grad = torch.empty((T, B, H), device="cuda")
    L = T.bit_length()

    def graph_ms(fn):
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(gr, stream=s, capture_error_mode="relaxed"):
                fn()
        torch.cuda.synchronize()
        return round(_time(gr.replay, reps=20), 4)

    res = {}
    for u in range(0, L):
        lv = (u, u + 1) if u + 1 <= L else (u, u)
        ws = api.workspace(api.scan_workspace_size(jac, "hybrid", levels=lv))
        res[f"u{lv[0]}_d{lv[1]}"] = graph_ms(
            lambda ws=ws, lv=lv: api.scan(jac, g, grad_h=grad, ws=ws, mode="hybrid", levels=lv))
    wsb = api.workspace(api.scan_workspace_size(jac, "blocked", 8, 8))
    res["blocked_8_8"] = graph_ms(lambda: api.scan(jac, g, grad_h=grad, ws=wsb, block0=8, block=8))
    return {"T": T, "B": B, "H": H, "leaves": "materialised J^T (DENSE)", "scan_ms_graph": res}


def sweep_train():
    """End-to-end training iterations (cuDNN forward + backward + Adam) on the
    paper's bitstream task, BPPSA backward vs torch autograd
    (cuDNN backward); same model, data and optimizer (paper_1907_10134_b200/train.py)."""
    import copy
    import torch
    import bppsa_workloads as W
    from paper_1907_10134_b200.train import AutogradTrainer, BitstreamRnn, BppsaTrainer
    out = {}
    for name, (T, B, H, C0, C) in {"c1": (1000, 16, 20, 8, 8), "c2": (30000, 16, 20, 16, 16)}.items():
        torch.manual_seed(0)
        ma = BitstreamRnn(H=H).cuda()
        mb = copy.deepcopy(ma)
        mb.rnn.flatten_parameters()
        ta, tb = BppsaTrainer(ma, lr=1e-5, block0=C0, block=C), AutogradTrainer(mb, lr=1e-5)
        x, y = W.bitstreams(T, B, seed=7)
        x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        res = {}
        for tag, tr in (("bppsa_iter_ms", ta), ("autograd_iter_ms", tb)):
            for _ in range(3):
                tr.step(x, y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                tr.step(x, y)
            e1.record()
            torch.cuda.synchronize()
            res[tag] = round(e0.elapsed_time(e1) / 10, 4)
        res["speedup"] = round(res["autograd_iter_ms"] / res["bppsa_iter_ms"], 2)
        out[name] = {"T": T, "B": B, "H": H, **res}
    # config 3: GRU on the IRMAS-shaped L set (F = 1034, C = 12), B = 64, lr 3e-4;
    # the BPPSA iteration includes the gate recompute "FO"
    from paper_1907_10134_b200.train import BppsaGruTrainer, IrmasGru
    torch.manual_seed(0)
    ma = IrmasGru(12).cuda()
    mb = copy.deepcopy(ma)
    mb.rnn.flatten_parameters()
    ta, tb = BppsaGruTrainer(ma, lr=3e-4, block0=16, block=16), AutogradTrainer(mb, lr=3e-4)
    x, y = W.irmas_like(1034, 12, 64, 7)
    x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    res = {}
    for tag, tr in (("bppsa_iter_ms", ta), ("autograd_iter_ms", tb)):
        for _ in range(3):
            tr.step(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            tr.step(x, y)
        e1.record()
        torch.cuda.synchronize()
        res[tag] = round(e0.elapsed_time(e1) / 10, 4)
    res["speedup"] = round(res["autograd_iter_ms"] / res["bppsa_iter_ms"], 2)
    out["c3_gru"] = {"F": 1034, "C": 12, "B": 64, "H": 20, **res}
    return out


def sweep_csr(api, pk=None):
    """Config 5: 97 %-pruned VGG-11 conv stack, B = 16, CSR transposed
    Jacobians.  Hybrid schedules (u, dl) vs the linear SpMV chain (0, 0)."""
    import torch
    import bppsa_workloads as W
    from paper_1907_10134_b200.vgg import CsrChain
    w = W.vgg11_workload(B=16, seed=0)
    relu_in = [torch.from_numpy(r[1]).cuda() for r in w["recs"] if r[0] == "relu"]
    pools = [torch.from_numpy(r[1]).cuda() for r in w["recs"] if r[0] == "pool"]
    chain = CsrChain(W.VGG11_CFG, w["weights"], relu_in, pools)
    seed = torch.from_numpy(w["g"]).cuda()
    res = {"B": 16, "n": chain.n, "nnz_total": int(sum(int(p[2][-1]) for p in chain.patterns))}
    for sched in ((0, 0), (1, 2), (2, 3)):
        t0 = time.perf_counter()
        plan = chain.plan(*sched)
        t_plan = time.perf_counter() - t0
        ws = api.workspace(plan.workspace_size(16, chain.batched))
        grads = [torch.empty((16, d), device="cuda") for d in plan.dims]
        run = lambda: api.csr_scan(plan, chain.data, chain.batched, seed, grads=grads, ws=ws)  # noqa: E731
        ms_eager = _time(run, reps=10)
        ms_graph = None                         # the launch-bound chains (44-59 kernels): CUDA-graph replay
        try:
            gr = torch.cuda.CUDAGraph()
            s_ = torch.cuda.Stream()
            s_.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_):
                run()
                torch.cuda.synchronize()
                with torch.cuda.graph(gr, stream=s_, capture_error_mode="relaxed"):
                    run()
            torch.cuda.synchronize()
            ms_graph = _time(gr.replay, reps=10)
            del gr
        except Exception as ex:  # noqa: BLE001
            ms_graph = f"capture failed: {ex}"[:120]
        ms = ms_graph if not isinstance(ms_graph, (str, type(None))) else ms_eager
        info = plan.info()
        steps = api.csr_plan_steps(plan)       # fig:prune_symbolic static FLOP analysis
        scan_st = [x for x in steps if x["phase"] != "bp"]
        bp_st = [x for x in steps if x["phase"] == "bp"]
        # HBM roofline: every planned contribution reads its two
        # (position, position) int32 plan entries (8 B) and gathers B floats of
        # each operand (2 x 4 B x B); every SpMV nnz reads its CSR index + value
        # (8 B) and B floats of the vector; every output element is written once
        Bb = 16
        out_el = sum(int(d) for d in plan.dims) * Bb
        c_bytes = info["contributions"] * (8 + 8 * Bb) + info["spmv_nnz"] * (8 + 4 * Bb) + out_el * 4
        hbm = pk["hbm_gbs"] if pk else 6527.0
        res_roof = {"bound": "hbm", "algorithmic_bytes": c_bytes,
                    "achieved_gbs": round(c_bytes / (ms * 1e-3) / 1e9, 1), "peak_gbs": hbm,
                    "frac": round(c_bytes / (ms * 1e-3) / 1e9 / hbm, 4)}
        res[f"u{sched[0]}_dl{sched[1]}"] = {
            "scan_ms": round(ms, 4), "scan_ms_eager": round(ms_eager, 4),
            "scan_ms_graph": ms_graph if isinstance(ms_graph, (str, type(None))) else round(ms_graph, 4),
            "plan_build_s": round(t_plan, 2), "roofline": res_roof,
            "contributions": info["contributions"], "spmv_nnz": info["spmv_nnz"],
            "kernels": info["kernels"], "ws_GB": round(ws.numel() / 1e9, 3),
            "flops_per_sample": {"bppsa_total": sum(x["flops"] for x in scan_st),
                                 "bppsa_critical_path": sum(x["flops"] for x in scan_st if x["critical"]),
                                 "bppsa_max_step": max(x["flops"] for x in scan_st),
                                 "bp_total": sum(x["flops"] for x in bp_st),
                                 "bp_max_step": max(x["flops"] for x in bp_st),
                                 "dense_equivalent_total": sum(x["dense_flops"] for x in scan_st)}}
        del ws, plan
        torch.cuda.empty_cache()
    # the paper's own schedule (up-sweep L0..L2, down-sweep L7..L10 = (3, 4)):
    # its contribution lists do not fit (9.1e10 pairs), so only the static FLOP
    # analysis of fig:prune_symbolic (host-only symbolic plan, no numeric scan)
    t0 = time.perf_counter()
    sym = api.csr_plan_create_symbolic(chain.patterns, 3, 4)
    t_sym = time.perf_counter() - t0
    steps = api.csr_plan_steps(sym)
    scan_st = [x for x in steps if x["phase"] != "bp"]
    bp_st = [x for x in steps if x["phase"] == "bp"]
    res["u3_dl4_symbolic"] = {
        "analysis_s": round(t_sym, 2), "contributions": sym.info()["contributions"],
        "steps": len(scan_st),
        "flops_per_sample": {"bppsa_total": sum(x["flops"] for x in scan_st),
                             "bppsa_critical_path": sum(x["flops"] for x in scan_st if x["critical"]),
                             "bppsa_max_step": max(x["flops"] for x in scan_st),
                             "bp_total": sum(x["flops"] for x in bp_st),
                             "bp_max_step": max(x["flops"] for x in bp_st),
                             "dense_equivalent_total": sum(x["dense_flops"] for x in scan_st)},
        "per_step": [{k: x[k] for k in ("kind", "phase", "level", "critical", "flops", "dense_flops")}
                     for x in scan_st]}
    del sym
    res["note"] = ("the paper's schedule (u, dl) = (3, 4) (P:472) needs 9.1e10 contribution pairs on this pruned "
                   "VGG-11: no numeric plan holds them, its static FLOP analysis is u3_dl4_symbolic "
                   "(bppsa_csr_plan_create_symbolic); (0, 0) is the linear scan = sequential BP with SpMVs")
    return res


# ----------------------------------------------------------------------------- reference arm
def host_cpu():
    """lscpu model name and logical CPUs of the host the oracle runs on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.TimeoutExpired):
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def _oracle_samples(args):
    """Worker of the OpenMP-style secondary: sequential BP of a slice of the samples."""
    import bppsa_workloads as W
    from oracle import bp
    from threadpoolctl import threadpool_limits
    Ts, b0, b1, seed = args
    with threadpool_limits(limits=1):
        w = W.rnn_workload(Ts, C4["B"], C4["H"], seed=seed)
        t0 = time.perf_counter()
        ref, _ = bp.bp_rnn(w.h[:, b0:b1], w.W_hh, w.g[b0:b1])
        bp.weight_grads_rnn(w.x[:, b0:b1], w.h[:, b0:b1], ref)
        return time.perf_counter() - t0


def oracle_sample(budget_s: float = 12.0, seed: int = 0):
    """Time the oracle (fp64 numpy sequential BP + weight grads) single-threaded
    on a T-sample of config 4 sized for ~budget_s, extrapolated linearly in T;
    secondary: the same sample split over the B samples across processes
    (sequential BP parallelises only across samples)."""
    from concurrent.futures import ProcessPoolExecutor
    from threadpoolctl import threadpool_limits
    import bppsa_workloads as W
    from oracle import bp
    T, B, H = C4["T"], C4["B"], C4["H"]
    Ts = 1 << 13
    with threadpool_limits(limits=1):
        while True:
            w = W.rnn_workload(Ts, B, H, seed=seed)
            t0 = time.perf_counter()
            ref, _ = bp.bp_rnn(w.h, w.W_hh, w.g)
            bp.weight_grads_rnn(w.x, w.h, ref)
            dt = time.perf_counter() - t0
            if dt * 4 > budget_s or Ts >= T:
                break
            Ts = min(T, Ts * 4)
    res = {"value": round(dt * 1e3 * T / Ts, 1), "unit": "ms", "cores": 1, "kind": "oracle",
           "sample": f"T={Ts} of {T} steps (B={B}, H={H}) fp64 sequential BP + weight grads, "
                     f"{dt:.2f} s measured single-threaded, extrapolated x{T // Ts} (linear in T)",
           "host": host_cpu()}
    P = max(1, min(B, os.cpu_count() or 1))
    try:
        step = -(-B // P)
        jobs = [(Ts, b0, min(B, b0 + step), seed) for b0 in range(0, B, step)]
        with ProcessPoolExecutor(max_workers=len(jobs)) as ex:
            times = list(ex.map(_oracle_samples, jobs))
        res["parallel_over_samples"] = {"value": round(max(times) * 1e3 * T / Ts, 1), "unit": "ms",
                                        "cores": len(jobs),
                                        "note": "the same sample, the B samples split over processes (one core "
                                                "each): the slowest process's oracle time, extrapolated likewise"}
    except Exception as ex:  # noqa: BLE001
        res["parallel_over_samples"] = {"error": str(ex)[:100]}
    return res


def run_reference(args):
    """The reference arm of this tier: the fp64 oracle (sequential BP + weight
    gradients) on the FULL C4 workload, once (steps = 1: ~30-60 s of one core;
    BPPSA_REF_T overrides T for quick checks and says so in `sample`)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    from threadpoolctl import threadpool_limits
    import bppsa_workloads as W
    from oracle import bp
    T = int(os.environ.get("BPPSA_REF_T", C4["T"]))
    B, H = C4["B"], C4["H"]
    w = W.rnn_workload(T, B, H, seed=args.seed)
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        ref, _ = bp.bp_rnn(w.h, w.W_hh, w.g)
        bp.weight_grads_rnn(w.x, w.h, ref)
        v = (time.perf_counter() - t0) * 1e3
    cb = {"value": round(v, 1), "unit": "ms", "cores": 1, "kind": "oracle",
          "sample": f"the full workload T={T} (B={B}, H={H}): fp64 sequential BP + weight grads, one run, "
                    f"single-threaded" + ("" if T == C4["T"] else f" (BPPSA_REF_T override; C4 has T={C4['T']})"),
          "host": host_cpu()}
    return {"metric": METRIC, "value": cb["value"], "unit": "ms", "n_gpus": world, "steps": 1,
            "warmup": 0, "ms_per_step": cb["value"], "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"C4: tanh RNN H=64 B=16 T={T} backward (sequential BP + weight grads)"},
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": "ms", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}


def run_dry(args):
    """BPPSA_BENCH_DRYRUN=1 (tests on CPU): the launcher / rendezvous /
    max-over-ranks path of the GPU arm with a fake per-rank time, over gloo."""
    import torch
    import torch.distributed as dist
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    ms = torch.tensor([1.0 + rank])
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
    return {"ms": float(ms[0]), "world": world}


def relaunch(args) -> int:
    """--gpus N > 1 without a torchrun environment: run this script as N ranks
    (one per GPU) through torch.distributed.run on 127.0.0.1."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--quick", action="store_true", help="skip e2e / baselines / sweep / cpu_baseline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world, rank, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        line = run_reference(args)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if os.environ.get("BPPSA_BENCH_DRYRUN"):
        r = run_dry(args)
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": r["ms"], "unit": "ms", "n_gpus": r["world"],
                              "steps": args.steps, "warmup": args.warmup, "dry_run": True}), flush=True)
        return
    r = run_ours(args)
    if rank != 0:
        return
    line = {"metric": METRIC, "value": round(r["ms"], 3), "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(r["ms"], 3), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded bitstreams x~Bernoulli(0.05+0.1c), torch-default init, fp32 forward "
                    "on the GPU (cuDNN, TF32 off); every rank keeps only its time shard)",
            "config": {"workload": "C4: tanh RNN, H=64, B=16, T=1048576 — full backward (fused leaves + "
                                   "blocked Blelloch scan + weight grads)",
                       "T": C4["T"], "B": C4["B"], "H": C4["H"], "block0": c4_block0(world), "block": C4_BLOCK,
                       "arithmetic": "fp32 results; level-0 fold and walk as exact s32 sums of int8 digit "
                                     "products (tcgen05 kind::i8), every rounding RN",
                       "parallelism": (f"contiguous time shards x{world}, "
                                       f"{os.environ.get('BPPSA_EXCHANGE', 'nccl')} carry exchange")
                                      if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (h = 4.3 GB, grad_h = 4.3 GB)"},
            "roofline": r["roofline"], "gpu_launches": r["launches"] * args.steps,
            "clocks": r["clocks"], "kernels_ms": [round(k, 4) for k in r["kernels_ms"]]}
    if world == 1 and not args.quick:
        line["e2e"] = r["e2e"]
        sb = r["sequential_bp"]
        sb["speedup_vs_gpu_linear"] = round(sb["gpu_linear_scan_ms"] / r["ms"], 2)
        sb["speedup_vs_cudnn"] = None if sb["cudnn_backward_ms"] is None else round(sb["cudnn_backward_ms"] / r["ms"], 2)
        line["sequential_bp"] = sb
        line["sweep"] = r["sweep"]
        line["sweep"]["affine_c4"] = r["affine"]
        line["cpu_baseline"] = oracle_sample()
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
