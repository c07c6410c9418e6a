"""Per-phase profile of the GPU tick.

The paper splits the serial simulator's time into Scheduler 2.2 %, Router
5.8 % and Neuron Block 91.7 %.  This reproduces the form of that split
for the two GPU kernels, plus the zero-spike "TrueNorth Ref." case:

  popcount kernel   per-phase clock64 sums over all CTAs (RANC_DEBUG_PHASES):
                    a1 scheduler read+clear, a2 input injection, spike words,
                    potential-load wait, a3-a6 fused neuron loop, store
  tensor-core path  busy cycles per role of CTA 0 (RANC_DEBUG_TIMELINE):
                    spike stage (a1, a2, operand expansion), MMA issue (a3),
                    epilogue (a4-a6); the roles overlap, so the largest one
                    sets the pace
  zero drive        config 5 with and without spikes, both kernels

  python tools/phase_profile.py [samples]      (prints markdown)
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
S = int(sys.argv[1]) if len(sys.argv) > 1 else 2000


def run(code, env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    return r.stdout, r.stderr


POPC = f"""
import sys; sys.path.insert(0, '.')
from paper_2404_16208_b200 import Simulator, OPT_KERNEL, OPT_STREAM
from workloads.gen import config3
net, inp = config3(S={S})
sim = Simulator(net); sim.set_option(OPT_KERNEL, 1); sim.set_option(OPT_STREAM, 1)
sim.load_inputs(inp).run(net.meta['T'])
"""
TC = f"""
import sys; sys.path.insert(0, '.')
from paper_2404_16208_b200 import Simulator, OPT_KERNEL
from workloads.gen import config3
net, inp = config3(S={max(S, 9472)})
sim = Simulator(net); sim.set_option(OPT_KERNEL, 2)
sim.load_inputs(inp).run(net.meta['T'])
"""
ZERO = """
import sys, torch; sys.path.insert(0, '.')
from paper_2404_16208_b200 import Simulator, OPT_KERNEL
from workloads.gen import config5
for drive in (True, False):
    net, inp = config5(S=64, T=60, grid=64, drive=drive)
    for k in (1, 2):
        st = torch.cuda.Stream()
        sim = Simulator(net, stream=st); sim.set_option(OPT_KERNEL, k); sim.load_inputs(inp)
        sim.run(10); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sim.reset(); a.record(st); sim.run(60); b.record(st); torch.cuda.synchronize()
        fired = int(sim.outputs().sum())
        print(f"drive={drive} kernel={k} ms_per_tick={a.elapsed_time(b) / 60:.4f} outputs={fired}")
        sim.close()
"""


def popc_table():
    _, err = run(POPC, {"RANC_DEBUG_PHASES": "1"})
    names = ["a1 scheduler read + clear", "a2 input injection", "spike words per piece",
             "potential load wait (TMA)", "a3-a6 integration + LIF + routing", "potential store (TMA)"]
    tot = [0] * 6
    n = 0
    for line in err.splitlines():
        m = re.match(r"phases t=(\d+) cycles .*: a1 (\d+) a2 (\d+) expand (\d+) potwait (\d+) a3-a6 (\d+) store (\d+)",
                     line)
        if m:
            vals = [int(x) for x in m.groups()[1:]]
            tot = [a + b for a, b in zip(tot, vals)]
            n += 1
    s = sum(tot) or 1
    out = [f"### popcount kernel (config 3, S = {S}, {n} ticks; CTA-cycles summed over all CTAs)", "",
           "| phase | share |", "|---|---|"]
    out += [f"| {nm} | {v / s * 100:.1f} % |" for nm, v in zip(names, tot)]
    return out


def tc_table():
    _, err = run(TC, {"RANC_DEBUG_TIMELINE": "1"})
    busy = {"spike stage (a1, a2, expansion)": 0, "MMA issue (a3)": 0, "epilogue warp 0 (a4-a6)": 0}
    ticks = 0
    rows = []
    for line in err.splitlines():
        if line.startswith("timeline t="):
            ticks += 1
            continue
        f = line.split()
        if len(f) == 17 and f[0].isdigit():
            v = [int(x) for x in f[1:]]
            if min(v[2], v[4], v[5], v[6], v[7], v[8], v[11]) < 0:
                continue
            rows.append(v)
            # columns: 2 FULL passed, 3 BEMPTY passed, 4 BFULL arrive, 14 synced
            busy["spike stage (a1, a2, expansion)"] += (v[14] - v[2]) + (v[4] - v[3])
            busy["MMA issue (a3)"] += v[7] - v[6]
            busy["epilogue warp 0 (a4-a6)"] += v[11] - v[8]
    out = [f"### tensor-core kernel (config 3, CTA 0, first 64 tiles of each of {ticks} ticks; busy cycles per role)",
           "", "| role | busy cycles per tile |", "|---|---|"]
    nt = max(1, len(rows))
    out += [f"| {k} | {v / nt:.0f} |" for k, v in busy.items()]
    return out


def zero_table():
    outp, err = run(ZERO, {})
    out = ["### zero-spike TrueNorth Ref. (config 5, 64x64 mesh, S = 64; P:218)", "",
           "| drive | kernel | ms / tick | output spikes |", "|---|---|---|---|"]
    for line in outp.splitlines():
        m = re.match(r"drive=(\w+) kernel=(\d) ms_per_tick=([\d.]+) outputs=(\d+)", line)
        if m:
            out.append(f"| {'driven' if m.group(1) == 'True' else 'zero'} | "
                       f"{'popcount' if m.group(2) == '1' else 'tensor core'} | {m.group(3)} | {m.group(4)} |")
    if len(out) == 4:
        out.append(f"| (failed: {err.strip()[-200:]}) | | | |")
    return out


if __name__ == "__main__":
    lines = ["## Per-phase profile (tools/phase_profile.py)", ""]
    for f in (popc_table, tc_table, zero_table):
        lines += f() + [""]
    print("\n".join(lines))
