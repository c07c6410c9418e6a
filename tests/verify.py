"""cmd_verify of SPEC: run the CUDA path once and the serial
oracle once on the same seeded workload and report the FIRST divergent record
(tick, sample, core, neuron) -- PASS iff every fired bit and every final
potential and class count agree ("one-to-one match between output
files").  Test infrastructure: imports oracle/."""
from __future__ import annotations

import numpy as np


def first_divergence(sim, net, inp, T):
    """`sim`: a Simulator with inputs loaded at tick 0 and SPIKE_RASTER tracing
    on; runs T ticks in ONE ranc_run_ticks call (so multi-tick launches are
    exercised) and compares the raster tick by tick with the oracle.  Returns
    None (PASS) or a dict locating the first divergent record."""
    from oracle.pyoracle import Oracle
    sim.run(T)
    raster = sim.raster()                    # [T][S][G][N]
    o = Oracle(net, inp)
    for t in range(T):
        o.run(1)
        ref = o.fired()
        if not np.array_equal(raster[t], ref):
            s, g, n = (int(v) for v in np.argwhere(raster[t] != ref)[0])
            return {"tick": t, "sample": s, "core": (g % net.grid_w, g // net.grid_w), "neuron": n,
                    "what": f"fired gpu={int(raster[t][s, g, n])} oracle={int(ref[s, g, n])}"}
    pot, ref = sim.potentials(), o.potentials()
    if not np.array_equal(pot, ref):
        s, g, n = (int(v) for v in np.argwhere(pot != ref)[0])
        return {"tick": T - 1, "sample": s, "core": (g % net.grid_w, g // net.grid_w), "neuron": n,
                "what": f"potential gpu={int(pot[s, g, n])} oracle={int(ref[s, g, n])}"}
    cnt, ref = sim.outputs(), o.counts()
    if not np.array_equal(cnt, ref):
        s, c = (int(v) for v in np.argwhere(cnt != ref)[0])
        return {"tick": T - 1, "sample": s, "core": None, "neuron": None,
                "what": f"class {c} count gpu={int(cnt[s, c])} oracle={int(ref[s, c])}"}
    return None


def verdict(div) -> str:
    if div is None:
        return "PASS"
    return (f"FAIL: first divergence at tick {div['tick']}, sample {div['sample']}, core {div['core']}, "
            f"neuron {div['neuron']}: {div['what']}")
