#!/usr/bin/env python
"""Summarise ncu reports for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep        # key metrics of a --set full capture
  python tools/ncu_summary.py launches gpurun_out/launches.csv    # per-kernel launch-time shares
  python tools/ncu_summary.py counters OUT.json REP...            # merge per-launch counters into OUT.json
      (REP named prof_<tag>_<workload>.ncu-rep; bench.py reads profiles/counters.json)
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
    "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Issued Instructions",
    "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction",
    "Eligible Warps Per Scheduler", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
       "l1tex__t_bytes_pipe_lsu_mem_global_op_red.sum", "lts__t_sectors_op_red.sum",
       "smsp__inst_executed.sum", "launch__registers_per_thread"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def full(rep):
    out = []
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))))
    h = rows[0]
    ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    idi = h.index("ID")
    seen = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if r[mi] in KEYS:
            seen[r[idi]][r[mi]] = f"{r[vi]} {r[ui]}".strip()
            names[r[idi]] = r[ki]
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    rh = raw[0]
    for r in raw[2:]:
        d = dict(zip(rh, r))
        rid = d.get("ID")
        for k in RAW:
            if k in d and d[k] not in ("", "n/a"):
                seen[rid][k] = f"{d[k]} {raw[1][rh.index(k)]}".strip()
    for rid, m in seen.items():
        out.append(f"## launch {rid}: {names.get(rid, '?')}")
        for k in KEYS + RAW:
            if k in m:
                out.append(f"- {k}: {m[k]}")
    return "\n".join(out)


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(j for j, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[i + 1:]:
        if len(r) > vi:
            d[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = ["| kernel | launches | mean ns | total share |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v):.0f} | {sum(v) / tot:.3f} |")
    return "\n".join(out)


def counters(out_json, reps):
    """Per (kernel, workload) counters of one launch: DRAM bytes, issued warp
    instructions, issue-slot utilisation, duration and SM clock."""
    import json
    import os
    import re
    db = json.load(open(out_json)) if os.path.exists(out_json) else {}
    for rep in reps:
        wl = re.sub(r"^prof_[^_]+_", "", os.path.basename(rep).replace(".ncu-rep", ""))
        raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
        if len(raw) < 3:
            continue
        h = raw[0]
        d = dict(zip(h, raw[2]))

        scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "hz": 1, "khz": 1e3, "mhz": 1e6,
                 "ghz": 1e9, "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "inst": 1, "%": 1}

        def f(k):   # value in base units (bytes, seconds, Hz)
            try:
                return float(d[k].replace(",", "")) * scale.get(raw[1][h.index(k)].strip().lower(), 1)
            except (KeyError, ValueError):
                return None
        name = d.get("Kernel Name", "?")
        kname = "tick_tc_kernel" if "tick_tc" in name else name.split("<")[0].split("(")[0].split("::")[-1]
        dur_ns = (f("gpu__time_duration.sum") or 0) * 1e9
        db.setdefault(kname, {})[wl] = {
            "kernel": name[:160], "dram_bytes": (f("dram__bytes_read.sum") or 0) + (f("dram__bytes_write.sum") or 0),
            "inst_executed": f("smsp__inst_executed.sum"),
            "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "duration_ns": dur_ns, "sm_hz": f("smsp__cycles_elapsed.avg.per_second")}
    json.dump(db, open(out_json, "w"), indent=1, sort_keys=True)
    return json.dumps(db, indent=1, sort_keys=True)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "counters":
        print(counters(path, sys.argv[3:]))
    else:
        print(full(path) if mode == "full" else launches(path))
