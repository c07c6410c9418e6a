#!/usr/bin/env python
"""Benchmark of the tick-accurate RANC core update on B200 (BASELINE.json).

Workload (N=1 line): config 3, the 512-core MNIST-shaped inference net,
10000 synthetic rate-coded samples, 19 ticks per sample.  With
N GPUs (torchrun) the 10000 samples are sharded over the ranks (strong
scaling); class counts are gathered once with NCCL at the end of each e2e
step.

A "step" = one pass of the whole hot path over the batch: state reset
(potentials <- initial, rings empty, counts 0) + 19 ticks of
scheduler read / input injection / integration / LIF / routing for every core
of every sample.  `value` times steps with the inputs already resident in
HBM; `e2e` times the public C-ABI path with host buffers: ranc_load_inputs
(H2D from pinned memory) + ranc_run_ticks + ranc_read_outputs (D2H), plus the
NCCL gather when N > 1.

`--impl reference` times the oracle (oracle/, plain serial C) on this box's
host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated core-ticks/sec & samples/sec, 512-core MNIST net, 1/2/4/8 B200"
UNIT = "samples/s"


def alg_bytes_per_core_tick(net):
    """potentials read + written (int16) and the scheduler row due
    now read + cleared; 1088 B at A = N = 256."""
    return 2 * 2 * net.neurons + 2 * 4 * ((net.axons + 31) // 32)


# name -> (builder(S) -> (net, inputs), default S, sharding at N > 1)
def _vmm(variant):
    def b(S):
        from workloads.gen import config4
        return config4(variant, S=S)
    return b


def _cfg(i, **kw):
    def b(S):
        from workloads import gen
        return getattr(gen, f"config{i}")(S=S, **kw)
    return b


WORKLOADS = {
    "config3": (_cfg(3), 10000, "samples"),
    "config1": (_cfg(1), 1, "samples"),
    "config2": (_cfg(2), 1000, "samples"),
    "vmm32": (_vmm("vmm32"), 1000, "samples"),
    "vmm256": (_vmm("vmm256"), 1000, "samples"),
    "vmm1024": (_vmm("vmm1024"), 1000, "samples"),
    "config5": (_cfg(5), 64, "cores"),
    # the same mesh with uniformly random (global) destinations
    "config5g": (_cfg(5, variant="global"), 64, "cores"),
    # TrueNorth Ref. as the paper ran it: every tick's work
    # on the 4096-core mesh "but with no spikes" (no drive, nothing fires)
    "config5z": (_cfg(5, drive=False), 64, "cores"),
    # streaming: the config-3 net fed one image per tick,
    # 10000 images in 10003 ticks, one sample (10010 ticks)
    "stream": (lambda S: __import__("workloads.gen", fromlist=["x"]).config3_stream(10000), 1, "samples"),
    # design-space sweep (f3): 8 variants of the config-3 net tiled into one
    # 32x128 grid, 1250 samples each (the config-3 work per step); value counts
    # variant-samples
    "sweep8": (lambda S: _sweep(8, S), 1250, "samples"),
    # config 3 with weights / leaks / thresholds x16 (13-bit weights, beyond
    # int8): the tensor-core wide-weight variant (two int8 operands)
    "config3w": (lambda S: __import__("workloads.gen", fromlist=["x"]).config3_wide(S=S), 10000, "samples"),
    # cores beyond 256 x 256 (configurable axons / neurons):
    # 4x4 mesh of 512-axon x 1024-neuron cores, tensor cores in neuron groups
    "bigcore": (lambda S: __import__("workloads.gen", fromlist=["x"]).bigcore(S=S), 4096, "samples"),
}


def _sweep(V, S):
    from paper_2404_16208_b200.sweep import tile_variants
    from workloads.gen import config3, sweep_variants
    net, inp = config3(S=S)
    return tile_variants(sweep_variants(net, V)), inp


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    ap.add_argument("--samples", type=int, default=0, help="samples (0 = the workload's default)")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--kernel", default="auto", choices=["auto", "popc", "tc"])
    ap.add_argument("--ring", default="auto", choices=["auto", "sample", "word", "history"],
                    help="tensor-core scheduler layout (RANC_OPT_RING_LAYOUT)")
    ap.add_argument("--operand", default="auto", choices=["auto", "folded", "compact"],
                    help="tensor-core integration operand (RANC_OPT_OPERAND)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-samples", type=int, default=0, help="oracle sample size (0 = auto)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------
# clocks sampled during the timed region
# ----------------------------------------------------------------------------
class Clocks:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, nm in enumerate(names):
                if len(r) > 5 + i and "Active" in r[5 + i] and "Not" not in r[5 + i]:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------------------
# oracle timing (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------
def _oracle_worker(args):
    idx, ticks = args
    from oracle.pyoracle import Oracle
    net, inp = _WORK["net"], _WORK["inp"]
    t0 = time.perf_counter()
    Oracle(net, inp.subset(idx)).run(ticks)
    return time.perf_counter() - t0


_WORK = {}


ORACLE_CORE_TICK_BUDGET = 60000   # core-ticks per worker process (~10-20 s of serial oracle)


def oracle_plan(net, n_samples, cores):
    """Bound the oracle's work: all T ticks of n_samples samples when that fits
    the per-core budget, else the first T' ticks (rate scaled to whole samples)."""
    T = net.meta["T"]
    per_worker = max(1, -(-n_samples // cores))
    ticks = min(T, max(1, ORACLE_CORE_TICK_BUDGET // (net.G * per_worker)))
    return ticks


def time_oracle(net, inp, n_samples, cores, ticks=None):
    """Run the oracle on n_samples samples spread over `cores` worker
    processes for `ticks` ticks (default: the workload's T); returns
    (samples/s, wall seconds, per-core samples/s), a sample counting as all T
    ticks (rate scaled by ticks/T when fewer ticks were run)."""
    import multiprocessing as mp
    from oracle import pyoracle
    pyoracle.build()
    _WORK["net"], _WORK["inp"] = net, inp
    T = net.meta["T"]
    ticks = ticks or T
    S = inp.num_samples
    pick = np.linspace(0, S - 1, n_samples).astype(int)
    chunks = [pick[i::cores] for i in range(cores)]
    chunks = [c for c in chunks if len(c)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(len(chunks)) as pool:
        per = pool.map(_oracle_worker, [(c, ticks) for c in chunks])
    wall = time.perf_counter() - t0
    frac = ticks / T
    per_core = statistics.median([len(c) * frac / p for c, p in zip(chunks, per)])
    return n_samples * frac / wall, wall, per_core


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------
def build_workload(args):
    builder, S0, mode = WORKLOADS[args.workload]
    if not args.samples:
        args.samples = S0
    net, inp = builder(args.samples)
    return net, inp, mode


def issue_roofline(ctr, launch_ms, peaks):
    """The second limit of the tick kernel (report both
    fractions): issued warp instructions of one launch (ncu
    smsp__inst_executed.sum, profiles/counters.json) over the live mean launch
    time, against 4 issue slots per clock per SM x 148 SMs at the max SM clock."""
    if not ctr or not ctr.get("inst_executed"):
        return None
    peak = 4 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6
    ach = ctr["inst_executed"] / (launch_ms / 1e3)
    return {"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-inst/s", "frac": ach / peak,
            "inst_per_launch": ctr["inst_executed"], "ncu_issue_active_pct": ctr.get("issue_active_pct"),
            "note": "ncu smsp__inst_executed.sum of one launch (profiles/counters.json) / mean launch time (CUDA "
                    "events); peak = 4 warp-instructions/clk/SM x 148 SMs x sm_max_mhz"}


def int_roofline(net, info, G_loc, S_local, tick_ms, kname):
    """Algorithmic integer work of the synaptic integration: ceil(A/32) x N
    AND+POPC words per (core, sample) per tick (DESIGN 7), against the
    measured POPC rate of this B200 (profiles/r01_int_peaks.json).  On the
    tensor-core path the same work runs as int8 MMAs (2 A N ops per
    core-tick) against the 4.5 POPS dense int8 nominal."""
    words = ((net.axons + 31) // 32) * net.neurons * G_loc * S_local
    try:
        popc = json.load(open(os.path.join(ROOT, "profiles", "r01_int_peaks.json")))["popc_per_s"]
    except Exception:
        popc = 4.5253e12
    if info["kernel"] == 1:
        ach = words / (tick_ms / 1e3)
        return {"bound": "alu (POPC)", "achieved": ach, "peak": popc, "unit": "POPC words/s", "frac": ach / popc,
                "note": "ceil(A/32) x N words per core-tick; peak = measured POPC rate (profiles/r01_int_peaks.json)"}
    ops = 2.0 * net.axons * net.neurons * G_loc * S_local
    ach = ops / (tick_ms / 1e3)
    return {"bound": "tensor (int8)", "achieved": ach, "peak": 4.5e15, "unit": "int8 op/s", "frac": ach / 4.5e15,
            "note": "2 A N MMA ops per core-tick (the integration as int8 MMAs); peak = 4.5 POPS dense int8 nominal"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    net, inp, _ = build_workload(args)
    T = net.meta["T"]
    cores = max(1, min(host_cores(), 32))
    n = args.cpu_samples or min(args.samples, 2 * cores)
    ticks = oracle_plan(net, n, cores)
    for _ in range(args.warmup):
        time_oracle(net, inp, max(1, cores // 2), cores, ticks)
    vals = []
    for _ in range(args.steps):
        v, wall, per_core = time_oracle(net, inp, n, cores, ticks)
        vals.append((v, wall, per_core))
    v = statistics.median([x[0] for x in vals])
    wall = statistics.median([x[1] for x in vals])
    per_core = statistics.median([x[2] for x in vals])
    G = net.G
    line = {
        "impl": "reference",
        "metric": METRIC if args.workload == "config3" else f"simulated core-ticks/sec & samples/sec, {net.name}",
        "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "i64", "data": "synthetic",
        "config": {"workload": net.name, "samples": args.samples, "ticks": T, "cores": G,
                   "step": f"oracle on {n} of the {args.samples} samples, {ticks} of {T} ticks"},
        "core_ticks_per_s": v * G * T,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{n} samples of {net.name}, {ticks} of {T} ticks (rate scaled to whole "
                                   f"samples), per step over {cores} processes",
                         "per_core_value": per_core},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_2404_16208_b200 import OPT_KERNEL, OPT_SAMPLE_TILE, Simulator
    from paper_2404_16208_b200 import build as pbuild
    if rank == 0:
        pbuild.build()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    net, inp_all, mode = build_workload(args)
    T = net.meta["T"]
    from paper_2404_16208_b200 import SHARD_CORES, SHARD_SAMPLES
    from paper_2404_16208_b200.dist import init_comm, shard_range
    core_sharded = mode == "cores" and world > 1
    lo, hi = (0, args.samples) if core_sharded else shard_range(args.samples, world, rank)
    inp = inp_all.slice(lo, hi)
    stream = torch.cuda.Stream(device=dev)
    sim = Simulator(net, device=local, stream=stream)
    if args.tile:
        sim.set_option(OPT_SAMPLE_TILE, args.tile)
    sim.set_option(OPT_KERNEL, {"auto": 0, "popc": 1, "tc": 2}[args.kernel])
    if args.ring != "auto":
        from paper_2404_16208_b200 import OPT_RING_LAYOUT
        sim.set_option(OPT_RING_LAYOUT, {"sample": 1, "word": 2, "history": 3}[args.ring])
    if args.operand != "auto":
        from paper_2404_16208_b200 import OPT_OPERAND
        sim.set_option(OPT_OPERAND, {"folded": 1, "compact": 2}[args.operand])
    if world > 1:
        init_comm(sim, world, rank, mode=SHARD_CORES if core_sharded else SHARD_SAMPLES)
    sim.load_inputs(inp)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---- device-resident timing -------------------------------------------
    for _ in range(args.warmup):
        sim.reset().run(T)
    barrier()
    launches0 = sim.info()["kernel_launches"]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk, torch.cuda.stream(stream):
        start.record(stream)
        for i in range(args.steps):
            sim.reset()
            ev[i][0].record(stream)
            sim.run(T)
            ev[i][1].record(stream)
        end.record(stream)
        barrier()
    launches = sim.info()["kernel_launches"] - launches0
    ms = start.elapsed_time(end)
    tick_ms = sum(a.elapsed_time(b) for a, b in ev) / (args.steps * T)
    t = torch.tensor([ms, tick_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, tick_ms = float(t[0]), float(t[1])
    ms_step = ms / args.steps
    V = int(net.meta.get("variants", 1))   # sweep batching: a sample of every variant per sample
    samples_s = args.samples * V / (ms_step / 1e3)
    core_ticks_s = args.samples / (ms_step / 1e3) * net.G * T   # net.G counts every variant's cores
    G_loc = sim.info()["cores_local"]

    # ---- end-to-end through the public API, host buffers --------------------
    pinned = torch.empty(inp.line_bits.size, dtype=torch.int32, pin_memory=True)
    pinned.numpy().view(np.uint32)[:] = inp.line_bits.reshape(-1)
    from workloads.netdef import Inputs
    hinp = Inputs(inp.num_samples, inp.num_input_ticks,
                  pinned.numpy().view(np.uint32).reshape(inp.line_bits.shape), inp.first_sample)
    counts = np.zeros((hi - lo, net.num_classes), np.int32)
    gather_n = args.samples
    for _ in range(max(1, args.warmup)):
        sim.load_inputs(hinp).run(T).outputs(counts)
        if world > 1:
            sim.gather_outputs(gather_n, 0, rank)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sim.load_inputs(hinp).run(T).outputs(counts)
        if world > 1:
            sim.gather_outputs(gather_n, 0, rank)
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t[0])
    e2e_val = args.samples * V * args.steps / e2e_s

    if rank == 0:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        hbm = peaks.get("hbm_gbs", 6650.0)   # (the recipe's fallback when MEASURED_PEAKS.json is absent)
        S_local = hi - lo
        bpt = alg_bytes_per_core_tick(net)
        alg_bytes = bpt * G_loc * S_local
        achieved = alg_bytes / (tick_ms / 1e3) / 1e9
        info = sim.info()
        kname = ("tick_tc_kernel" if info["kernel"] == 2 else
                 "tick_stream_kernel" if launches == args.steps else "tick_popc_kernel")
        # per-launch ncu counters of this kernel on this workload (profiles/counters.json,
        # tools/profile_all.sh + tools/ncu_summary.py counters), when profiled
        ctr = None
        cpath = os.path.join(ROOT, "profiles", "counters.json")
        wl_key = args.workload + ("_popc" if args.kernel == "popc" else "")
        if os.path.exists(cpath) and S_local == args.samples:
            for kn, per_wl in json.load(open(cpath)).items():
                if kn.startswith(kname[:12]) and wl_key in per_wl:
                    ctr = per_wl[wl_key]
        # a multi-tick (cooperative) launch runs all T ticks of a step
        ticks_per_launch = T if launches == args.steps else 1
        traffic = ctr["dram_bytes"] / ticks_per_launch if ctr else None
        state_gb = (2 * net.neurons * net.G + 4 * info["ring_rows"] * info["ring_words"] * net.G) * args.samples / 1e9
        line = {
            "metric": METRIC if args.workload == "config3" else f"simulated core-ticks/sec & samples/sec, {net.name}",
            "value": samples_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "i32", "data": "synthetic",
            "config": {"workload": net.name, "samples": args.samples, "ticks": T, "cores": net.G,
                       "axons": net.axons, "neurons": net.neurons,
                       "parallelism": f"core-sharded x{world} (row bands, per-tick NCCL exchange)" if core_sharded
                       else f"sample-sharded dp{world}",
                       "l2": (f"state {state_gb:.2f} GB exceeds the 126 MB L2; no flush needed" if state_gb > 0.126
                              else f"state {state_gb * 1e3:.1f} MB fits in L2 (latency-bound workload)"),
                       "sample_tile": info["sample_tile"], "pieces": info["pieces"],
                       "ring_layout": {1: "sample-major", 2: "word-major", 3: "history"}.get(info["ring_layout"]),
                       "operand": {1: "folded", 2: "compact"}.get(info["operand"]),
                       "kernel": ("tcgen05 kind::i8" if info["kernel"] == 2 else
                                  "popcount, streaming (one cooperative launch per run)" if launches == args.steps
                                  else "popcount")},
            "core_ticks_per_s": core_ticks_s,
            "ticks_per_s": T / (ms_step / 1e3),
            "tick_kernel_ms": tick_ms,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "kernel": kname,
                         "note": f"{bpt} B/core-tick x {G_loc} cores x {S_local} samples per "
                                 "launch / mean launch time (CUDA events on the launch stream); peak = "
                                 "MEASURED_PEAKS.json hbm_gbs; traffic = ncu dram bytes per launch "
                                 "(profiles/traffic.json)"},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(inp.line_bits.nbytes),
                    "d2h_bytes_per_step": int(counts.nbytes)},
            "clocks": clk.summary(),
            "roofline_issue": issue_roofline(ctr, tick_ms * ticks_per_launch, peaks),
            "roofline_int": int_roofline(net, info, G_loc, S_local, tick_ms, kname),
        }
        if not args.no_cpu_baseline and world == 1:
            cores = max(1, min(host_cores(), 32))
            n = args.cpu_samples or min(args.samples, 8 * cores)   # ~10-20 s of oracle work
            ticks = oracle_plan(net, n, cores)
            v, wall, per_core = time_oracle(net, inp_all, n, cores, ticks)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": f"{n} of the {args.samples} samples, {ticks} of {T} ticks (rate scaled "
                                              f"to whole samples), over {cores} processes ({wall:.1f} s)",
                                    "per_core_value": per_core}
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` outside torchrun: start the N ranks (one
    process per GPU) with torch.distributed.run on this node and return its
    exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, max(world, args.gpus))
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
