"""GPU parity at the BENCHMARKED shapes ("a one-to-one match between
output files across all applications"), in the launch configurations
bench.py times, plus the configurable envelope of the ABI.

The oracle cannot replay 10000 x 512 cores or 64 x 4096 cores in seconds, so
the GPU runs the whole workload and records the per-(tick, sample) state
digest (potentials, fired neurons and integrated axon spikes
of every core); the oracle replays a sample slice -- one worker process per
sample, samples are independent (G14, pinned by batch composition P9) --
and the digests of those samples must agree at EVERY tick.
"""
import numpy as np
import pytest

from oracle_pool import oracle_digests
from workloads.gen import VMM_VARIANTS, config3, config5, envelope_case, vmm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ranc():
    from paper_2404_16208_b200 import build
    build.build()
    import paper_2404_16208_b200 as m
    return m


def gpu_digests(ranc, net, inp, T, kernel=0, ring=0):
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_KERNEL, kernel)
    sim.set_option(ranc.OPT_RING_LAYOUT, ring)
    sim.set_trace(ranc.TRACE_STATE_DIGEST)
    sim.load_inputs(inp).run(T)
    info = sim.info()
    d, cnt, pot = sim.digests(), sim.outputs(), sim.potentials()
    sim.close()
    return d, cnt, pot, info


def check_digests(name, got, ref, idx):
    for t in range(ref.shape[0]):
        bad = np.flatnonzero(got[t, idx] != ref[t])
        assert bad.size == 0, f"{name}: tick {t}, sample {idx[bad[0]]}: digest differs from the oracle"


def test_config3_one_sample_per_tile_every_tick(ranc):
    """Config 3 as benchmarked (10000 samples, 19 ticks, the automatic kernel:
    tcgen05, sample-major rings, per-tick launches): one sample from EVERY
    64-sample tile (157 samples, incl. the ragged last tile), per-tick
    digests against the oracle, plus final potentials and class counts."""
    net, inp = config3(S=10000)
    T = net.meta["T"]
    d, cnt, pot, info = gpu_digests(ranc, net, inp, T)
    assert info["kernel"] == 2 and info["ring_layout"] == 1
    nT = (10000 + 63) // 64
    idx = np.array([min(64 * k + (k * 37) % 64, 9999) for k in range(nT)])
    (ref_d, ref_c, ref_p), = oracle_digests([(net, inp, idx, T)])
    check_digests("config3", d, ref_d, idx)
    assert np.array_equal(cnt[idx], ref_c)
    assert np.array_equal(pot[idx], ref_p)
    assert cnt.sum() > 0


@pytest.mark.parametrize("ring", [0, 2])
@pytest.mark.parametrize("variant", ["local", "global"])
def test_config5_full_mesh_every_tick(ranc, variant, ring):
    """Config 5 as benchmarked: the 64x64 mesh (4096 cores, D = 15), S = 64,
    per-tick launches -- the automatic layout (history scheduler, compact
    operand expanded on chip) and the word-major ring (folded operand); 100
    ticks, samples 0 and 63 (the first and last lane of the 64-sample tile)
    replayed by the oracle."""
    T = 100
    net, inp = config5(S=64, T=T, variant=variant)
    d, cnt, pot, info = gpu_digests(ranc, net, inp, T, ring=ring)
    assert info["kernel"] == 2
    assert (info["ring_layout"], info["operand"]) == ((3, 2) if ring == 0 else (2, 1))
    idx = np.array([0, 63])
    (ref_d, ref_c, ref_p), = oracle_digests([(net, inp, idx, T)])
    check_digests(f"config5-{variant}", d, ref_d, idx)
    assert np.array_equal(pot[idx], ref_p)
    assert np.array_equal(cnt[idx], ref_c)


@pytest.mark.parametrize("ring", [0, 1])
def test_vmm1024_closed_form_full_batch(ranc, ring):
    """VMM-1024 as benchmarked (256 cores on a 16x16 grid, S = 1000, drained;
    the automatic layout -- the history scheduler -- and sample-major rings):
    the class counts of every sample equal M+ x and M- x (P6, numpy)."""
    net, inp = vmm(S=1000, seed=1004, **VMM_VARIANTS["vmm1024"])
    M, X = net.meta["M"], net.meta["X"]
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_RING_LAYOUT, ring)
    sim.load_inputs(inp).run(net.meta["T"])
    cnt = sim.outputs()
    assert sim.info()["kernel"] == 2
    assert sim.info()["ring_layout"] == (3 if ring == 0 else 1)
    sim.close()
    assert np.array_equal(cnt[:, 0::2], X @ np.maximum(M, 0).T)
    assert np.array_equal(cnt[:, 1::2], X @ np.maximum(-M, 0).T)


@pytest.mark.parametrize("seed", range(32))
@pytest.mark.parametrize("kernel", ["popc", "tc"])
def test_envelope_every_tick(ranc, oracle_mod, seed, kernel):
    """A, N up to 1024, full-range 13..16-bit weights, pb down to 2: full
    state against the oracle after every tick.  Beyond the tensor-core
    envelope the "tc" case is skipped (RANC_E_CONFIG)."""
    net, inp = envelope_case(seed)
    sim = ranc.Simulator(net)
    try:
        sim.set_option(ranc.OPT_KERNEL, 1 if kernel == "popc" else 2)
    except ranc.RancError as e:
        sim.close()
        assert e.code == "RANC_E_CONFIG"
        pytest.skip("outside the tensor-core envelope")
    sim.set_trace(ranc.TRACE_SPIKE_RASTER)
    sim.load_inputs(inp)
    o = oracle_mod.Oracle(net, inp)
    for t in range(10):
        sim.run(1)
        o.run(1)
        where = f"{net.name} tick {t}"
        assert np.array_equal(sim.potentials(), o.potentials()), where + " potentials"
        assert np.array_equal(sim.raster()[0], o.fired()), where + " fired"
        assert np.array_equal(sim.pending(), o.pending()), where + " pending"
        assert np.array_equal(sim.outputs(), o.counts()), where + " counts"
    sim.close()


def test_envelope_multi_tick_calls(ranc, oracle_mod):
    """The same envelope through one ranc_run_ticks call per run (streaming /
    multi-item cooperative launches where eligible)."""
    for seed in range(32):
        net, inp = envelope_case(seed)
        sim = ranc.Simulator(net)
        sim.load_inputs(inp).run(10)
        o = oracle_mod.Oracle(net, inp).run(10)
        assert np.array_equal(sim.potentials(), o.potentials()), net.name
        assert np.array_equal(sim.outputs(), o.counts()), net.name
        assert np.array_equal(sim.pending(), o.pending()), net.name
        sim.close()


@pytest.mark.parametrize("kernel", ["tc", "popc"])
@pytest.mark.parametrize("A,N", [(512, 1024), (256, 1024), (300, 257), (512, 128), (1024, 1024), (700, 300),
                                 (1024, 128)])
def test_bigcore_every_tick(ranc, oracle_mod, kernel, A, N):
    """Cores beyond 256 x 256: on the tensor cores they run as
    neuron groups (256 rows when A <= 256 and Npad % 256 == 0, else 128);
    full state against the oracle after every tick, 70 samples (a ragged
    second tile)."""
    from workloads.gen import bigcore
    net, inp = bigcore(S=70, T=8, A=A, N=N, grid=2)
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_KERNEL, 2 if kernel == "tc" else 1)
    sim.set_trace(ranc.TRACE_SPIKE_RASTER)
    sim.load_inputs(inp)
    assert sim.info()["kernel"] == (2 if kernel == "tc" else 1)
    o = oracle_mod.Oracle(net, inp)
    for t in range(8):
        sim.run(1)
        o.run(1)
        where = f"{net.name} tick {t}"
        assert np.array_equal(sim.potentials(), o.potentials()), where + " potentials"
        assert np.array_equal(sim.raster()[0], o.fired()), where + " fired"
        assert np.array_equal(sim.pending(), o.pending()), where + " pending"
        assert np.array_equal(sim.outputs(), o.counts()), where + " counts"
    sim.close()


def test_bigcore_full_size_digests(ranc):
    """The bench's big-core workload (16 cores of 512 axons x 1024 neurons,
    4096 samples, 20 ticks) on the tensor cores in neuron groups: per-tick
    digests of one sample from each of 16 tiles spread over the batch."""
    from workloads.gen import bigcore
    net, inp = bigcore()
    T = net.meta["T"]
    d, cnt, pot, info = gpu_digests(ranc, net, inp, T)
    assert info["kernel"] == 2
    idx = np.array([64 * k * 4 + (k * 13) % 64 for k in range(16)])
    (ref_d, ref_c, ref_p), = oracle_digests([(net, inp, idx, T)])
    check_digests("bigcore", d, ref_d, idx)
    assert np.array_equal(cnt[idx], ref_c)
    assert np.array_equal(pot[idx], ref_p)
