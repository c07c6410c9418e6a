"""Smoke-size runs of every kernel variant, for compute-sanitizer
(memcheck / synccheck / initcheck / racecheck):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [variant ...]

Each variant is checked against the oracle at the end (bit-exact), so a run
that the sanitizer lets through is also a parity run.  Variants: popc (per-tick
popcount launches), popc_stream (cooperative one-launch streaming kernel),
tc (per-tick tcgen05 kernel, sample-major rings), tc_wm (word-major rings),
tc_multi (cooperative multi-tick tcgen05 launch, neighbourhood barrier),
tc_wide (16-bit weights: u8/s8 split), tc_pull (history scheduler with the
compact operand), tc_pull_fold (history scheduler, folded operand), tc_comp
(compact operand, sample-major rings, input injection), tc_grp (neuron
groups), loopback (core-sharded group of 2 with the exchange kernels), digest.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(argv):
    from oracle.pyoracle import Oracle
    import paper_2404_16208_b200 as r
    from workloads.gen import config2, config5

    def check(sim, net, inp, T, what):
        o = Oracle(net, inp).run(T)
        assert np.array_equal(sim.potentials(), o.potentials()), what
        assert np.array_equal(sim.outputs(), o.counts()), what
        assert np.array_equal(sim.pending(), o.pending()), what
        print(f"ok {what}: kernel={sim.info()['kernel']} ring={sim.info()['ring_layout']} "
              f"launches={sim.info()['kernel_launches']}", flush=True)

    def run(net, inp, T, kernel, stream, ring=0, what="", trace=0, operand=0):
        sim = r.Simulator(net)
        sim.set_option(r.OPT_KERNEL, kernel)
        sim.set_option(r.OPT_STREAM, stream)
        if kernel == 2:
            sim.set_option(r.OPT_RING_LAYOUT, ring)
            sim.set_option(r.OPT_OPERAND, operand)
        if trace:
            sim.set_trace(trace)
        sim.load_inputs(inp).run(T)
        check(sim, net, inp, T, what)
        sim.close()

    variants = argv or ["popc", "popc_stream", "tc", "tc_wm", "tc_multi", "tc_wide", "tc_pull", "tc_pull_fold",
                        "tc_comp", "tc_grp", "loopback", "digest"]
    net2, inp2 = config2(S=70)
    T2 = net2.meta["T"]
    mesh, mesh_in = config5(S=3, T=6, grid=6)
    for v in variants:
        if v == "popc":
            run(net2, inp2, 6, 1, 1, what=v)
        elif v == "popc_stream":
            run(net2, inp2, T2, 1, 2, what=v)
        elif v == "tc":
            run(net2, inp2, 6, 2, 1, ring=1, what=v)
        elif v == "tc_wm":
            run(mesh, mesh_in, 6, 2, 1, ring=2, what=v)
        elif v == "tc_multi":
            run(net2, inp2, T2, 2, 2, what=v)
            run(mesh, mesh_in, 6, 2, 2, ring=2, what=v + "_wm")
        elif v == "tc_wide":
            w = mesh.copy()
            for f in ("weight", "leak", "pos_threshold", "neg_threshold", "reset_potential", "initial_potential"):
                setattr(w, f, getattr(w, f) * 100)
            for f in ("weight_bits", "leak_bits", "threshold_bits", "reset_bits"):
                setattr(w, f, getattr(w, f) + 7)
            run(w, mesh_in, 6, 2, 1, ring=2, what=v)
        elif v == "tc_pull":
            run(mesh, mesh_in, 6, 2, 1, ring=3, what=v, operand=2)
        elif v == "tc_pull_fold":
            run(mesh, mesh_in, 6, 2, 1, ring=3, what=v, operand=1)
        elif v == "tc_comp":
            run(net2, inp2, 6, 2, 1, ring=1, what=v, operand=2)
        elif v == "tc_grp":
            from workloads.gen import bigcore
            for A, N in ((512, 1024), (256, 512)):
                big, big_in = bigcore(S=70, T=4, A=A, N=N, grid=2)
                run(big, big_in, 4, 2, 1, what=f"{v}_A{A}_N{N}")
        elif v == "loopback":
            sims = [r.Simulator(mesh) for _ in range(2)]
            for s in sims:
                s.set_option(r.OPT_KERNEL, 2)
            r.Simulator.init_loopback(sims)
            for s in sims:
                s.load_inputs(mesh_in)
            r.Simulator.run_loopback(sims, 6)
            o = Oracle(mesh, mesh_in).run(6)
            got = np.concatenate([s.potentials() for s in sims], axis=1)
            assert np.array_equal(got, o.potentials()), v
            print(f"ok {v}", flush=True)
            for s in sims:
                s.close()
        elif v == "digest":
            run(net2, inp2, 4, 2, 1, ring=1, what=v, trace=r.TRACE_STATE_DIGEST | r.TRACE_OUTPUT_EVENTS)
        else:
            raise SystemExit(f"unknown variant {v}")


if __name__ == "__main__":
    main(sys.argv[1:])
