"""Sweep batching: V variants tiled into one network compute,
block by block, what each variant computes alone.  Pinned with the oracle on
CPU (the tiling is host-side table building; the GPU check is in
test_gpu_parity.py)."""
import dataclasses

import numpy as np
import pytest

from paper_2404_16208_b200.sweep import split_counts, split_potentials, tile_variants
from workloads.gen import config1, config2, corpus_case, sweep_variants


def _check(oracle_mod, variants, inp, T):
    tiled = tile_variants(variants)
    V, G, C = len(variants), variants[0].G, variants[0].num_classes
    ot = oracle_mod.Oracle(tiled, inp).run(T)
    cnt = split_counts(ot.counts(), V, C)
    pot = split_potentials(ot.potentials(), V, G)
    for v, net in enumerate(variants):
        o = oracle_mod.Oracle(net, inp).run(T)
        assert np.array_equal(cnt[:, v], o.counts()), f"variant {v} counts"
        assert np.array_equal(pot[:, v], o.potentials()), f"variant {v} potentials"
    return tiled


def test_sweep_config2_variants(oracle_mod):
    net, inp = config2(S=6)
    variants = sweep_variants(net, 4)
    tiled = _check(oracle_mod, variants, inp, net.meta["T"])
    assert tiled.grid_h == 4 * net.grid_h and tiled.num_classes == 4 * net.num_classes
    # the variants really differ
    cnts = [oracle_mod.Oracle(v, inp).run(net.meta["T"]).counts() for v in variants]
    assert any(not np.array_equal(cnts[0], c) for c in cnts[1:])


def test_sweep_self_routing_core(oracle_mod):
    net, inp = config1(T=40)
    _check(oracle_mod, sweep_variants(net, 3), inp, 40)


@pytest.mark.parametrize("seed", range(6))
def test_sweep_mixed_types_and_delays(oracle_mod, seed):
    a, inp = corpus_case(seed)
    b, _ = corpus_case(seed + 100)
    # second variant: the first one's shape with another draw of parameters
    # where shapes agree; otherwise just a reparametrised copy of the first
    if (b.grid_w, b.grid_h, b.axons, b.neurons, b.num_classes, b.num_lines, b.potential_bits) != \
            (a.grid_w, a.grid_h, a.axons, a.neurons, a.num_classes, a.num_lines, a.potential_bits):
        b = sweep_variants(a, 2, seed=seed)[1]
    _check(oracle_mod, [a, b, a], inp, 15)


def test_sweep_rejects_different_potential_bits():
    net, _ = config2(S=1)
    other = dataclasses.replace(net, potential_bits=12)
    with pytest.raises(ValueError, match="potential_bits"):
        tile_variants([net, other])
