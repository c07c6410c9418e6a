"""P6 (VMM closed form) and P9 (relabeling, batch composition, resumability)
pins of the oracle.  CPU only."""
import numpy as np
import pytest

from nets import permute_axons, permute_neurons
from workloads.gen import config2, corpus_case, vmm
from workloads.rng import substream


@pytest.mark.parametrize("n,m,Mmax,Xmax,block_in", [(12, 12, 15, 15, None),
                                                    (16, 10, 7, 5, 8),
                                                    (40, 24, 3, 7, 16)])
def test_vmm_closed_form(oracle_mod, n, m, Mmax, Xmax, block_in):
    # P6: counting network; after draining, count(j+) = (M+ x)_j and
    # count(j-) = (M- x)_j, so y = M x exactly.  Pinned by numpy matmul.
    net, inp = vmm(n, m, Mmax, Xmax, S=6, seed=5, block_in=block_in)
    M, X = net.meta["M"], net.meta["X"]
    o = oracle_mod.Oracle(net, inp).run(net.meta["T"])
    cnt = o.counts()
    yp = X @ np.maximum(M, 0).T
    yn = X @ np.maximum(-M, 0).T
    assert np.array_equal(cnt[:, 0::2], yp)
    assert np.array_equal(cnt[:, 1::2], yn)
    assert np.array_equal(cnt[:, 0::2] - cnt[:, 1::2], X @ M.T)
    if block_in:
        assert net.meta["two_layer"]


def _perms(seed, G, n):
    r = substream(seed, "perm")
    return [r.permutation(n) for _ in range(G)]


@pytest.mark.parametrize("seed", [1, 2, 5, 9])
def test_axon_relabeling_invariance(oracle_mod, seed):
    # P9: relabeling axons (with crossbar, types, lines and routes rewritten)
    # leaves potentials, counts and events unchanged; pending is permuted.
    net, inp = corpus_case(seed)
    inp = inp.slice(0, min(inp.num_samples, 4))
    perms = _perms(seed, net.G, net.axons)
    net2 = permute_axons(net, perms)
    a = oracle_mod.Oracle(net, inp).run(12)
    b = oracle_mod.Oracle(net2, inp).run(12)
    assert np.array_equal(a.potentials(), b.potentials())
    assert np.array_equal(a.events(), b.events())
    pa, pb = a.pending(), b.pending()
    for c in range(net.G):
        assert np.array_equal(pb[:, c][..., perms[c]], pa[:, c])


@pytest.mark.parametrize("seed", [1, 4, 7])
def test_neuron_relabeling_invariance(oracle_mod, seed):
    net, inp = corpus_case(seed)
    inp = inp.slice(0, min(inp.num_samples, 4))
    perms = _perms(seed + 100, net.G, net.neurons)
    net2 = permute_neurons(net, perms)
    a = oracle_mod.Oracle(net, inp).run(12)
    b = oracle_mod.Oracle(net2, inp).run(12)
    pa, pb = a.potentials(), b.potentials()
    for c in range(net.G):
        assert np.array_equal(pb[:, c][:, perms[c]], pa[:, c])
    assert np.array_equal(a.counts(), b.counts())
    assert np.array_equal(a.pending(), b.pending())


def test_batch_composition_and_resume(oracle_mod):
    # samples are independent (G14): any subset simulates identically; and
    # run(a) + run(b) == run(a + b).
    net, inp = config2(S=12)
    full = oracle_mod.Oracle(net, inp).run(17)
    sub = oracle_mod.Oracle(net, inp.subset([3, 7, 11])).run(17)
    assert np.array_equal(full.potentials()[[3, 7, 11]], sub.potentials())
    assert np.array_equal(full.counts()[[3, 7, 11]], sub.counts())
    split = oracle_mod.Oracle(net, inp).run(5).run(12)
    assert np.array_equal(split.potentials(), full.potentials())
    assert np.array_equal(split.events(), full.events())
