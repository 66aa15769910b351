#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (tracked).

  python scripts/summarize_ncu.py ROUND LAUNCHES_CSV|- [REPORT.ncu-rep KERNEL_KEY] ...

Writes profiles/<ROUND>_launches.md (per-kernel share of the step from the
`--metrics gpu__time_duration.sum` launch list), profiles/<ROUND>_<key>_ncu.md
(key counters of the `--set full` capture) and merges the per-launch DRAM
traffic into profiles/ncu_traffic.json (read by bench.py's roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}


def launches(path, rnd):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in data:
        agg[r[ki].split("(")[0].replace("void ", "")[:70]].append(float(r[vi].replace(",", "")) * UNIT[r[ui]])
    ours = {k: v for k, v in agg.items() if k.startswith("bppsa::")}
    tot = sum(sum(v) for v in ours.values())
    out = [f"# {rnd}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)", "",
           f"source: {os.path.basename(path)}; cold-cache serialised launches — compare SHARES, not absolutes.",
           "Shares are of the library's (bppsa::) kernels; the rest is the bench's input build (cuDNN forward).",
           "", "| kernel | launches | avg ms | total ms | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        sh = f"{sum(v) / tot:.1%}" if k in ours else "(input build)"
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.4f} | {sum(v):.3f} | {sh} |")
    open(os.path.join(PROF, f"{rnd}_launches.md"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def report(path, key, rnd):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    name = d.get("Kernel Name", ("?", ""))[0]
    stalls = []
    for h, (v, _) in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    tot = sum(s for s, _ in stalls) or 1.0
    lines = [f"# {rnd}: `ncu --set full` of {key}", "", f"kernel: `{name[:160]}`", "",
             "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in d:
            lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
    lines += ["", "Warp stall samples (share):", ""]
    lines += [f"- {n}: {s / tot:.1%}" for s, n in stalls[:8]]
    open(os.path.join(PROF, f"{rnd}_{key}_ncu.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

    def num(k):
        v, u = d[k]
        f = float(v.replace(",", ""))
        return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)

    tj = os.path.join(PROF, "ncu_traffic.json")
    t = json.load(open(tj)) if os.path.exists(tj) else {}
    t[key] = {"dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
              "round": rnd, "kernel": name[:160],
              "duration_ms_under_ncu": float(d["gpu__time_duration.sum"][0].replace(",", "")) *
              UNIT.get(d["gpu__time_duration.sum"][1], 1.0)}
    json.dump(t, open(tj, "w"), indent=1)


if __name__ == "__main__":
    rnd = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    if sys.argv[2] != "-":
        launches(sys.argv[2], rnd)
    rest = sys.argv[3:]
    for i in range(0, len(rest), 2):
        report(rest[i], rest[i + 1], rnd)
