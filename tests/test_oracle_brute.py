"""P7: the oracle against an independent dense NumPy brute force on random
tiny meshes, full state after every tick (SPEC acceptance 2)."""
import numpy as np
import pytest

import brute
from workloads.gen import corpus_case, tiny_case

N_SEEDS = 1000


def compare(oracle_mod, net, inp, T):
    states, ev = brute.run(net, inp, T)
    o = oracle_mod.Oracle(net, inp)
    for t in range(T):
        o.run(1)
        st = states[t]
        assert np.array_equal(o.potentials(), st["pot"]), f"pot tick {t}"
        assert np.array_equal(o.fired().astype(bool), st["fired"]), f"fired tick {t}"
        assert np.array_equal(o.pending().astype(bool), st["pending"]), f"pending tick {t}"
        assert np.array_equal(o.counts(), st["counts"]), f"counts tick {t}"
    assert np.array_equal(o.events(), ev)


@pytest.mark.parametrize("block", range(10))
def test_tiny_meshes_vs_brute(oracle_mod, block):
    per = N_SEEDS // 10
    for seed in range(block * per, (block + 1) * per):
        net, inp = tiny_case(seed)
        compare(oracle_mod, net, inp, 20)


@pytest.mark.parametrize("seed", range(6))
def test_corpus_vs_brute(oracle_mod, seed):
    net, inp = corpus_case(seed)
    if inp.num_samples > 8:
        inp = inp.slice(0, 8)
    compare(oracle_mod, net, inp, 14)


def test_brute_is_not_trivially_silent():
    # the corpus must exercise spikes, routes, outputs and saturation
    fired = routed = outs = 0
    for seed in range(50):
        net, inp = tiny_case(seed)
        states, ev = brute.run(net, inp, 20)
        fired += sum(int(s["fired"].sum()) for s in states)
        routed += sum(int(s["pending"].sum()) for s in states)
        outs += len(ev)
    assert fired > 100 and routed > 100 and outs > 50
