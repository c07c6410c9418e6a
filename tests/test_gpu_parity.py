"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit-exact
for every potential, pending spike, fired bit, output event and class count
("a one-to-one match between output files")."""
import numpy as np
import pytest

from workloads.gen import (config1, config2, config3, config3_stream, config4, config5, corpus_case, sweep_variants,
                           tiny_case, vmm)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ranc():
    from paper_2404_16208_b200 import build
    build.build()
    import paper_2404_16208_b200 as m
    return m


# "tc": tensor-core kernel, sample-major scheduler rings; "tc_wm": word-major
# rings (RANC_OPT_RING_LAYOUT = 2); "tc_gather": word-major rings and the
# per-tick input-run gather instead of the load-time input decode
# (RANC_OPT_INPUT_DECODE = 0); "tc_pull": the history scheduler (layout 3:
# destination-ordered fired-bit history).  Operand: "tc" forces the folded
# Wfold (RANC_OPT_OPERAND = 1), "tc_comp" the compact operand expanded on
# chip (2); the others take the automatic choice (compact for the few-tile
# batches of these tests when the network is eligible).
KERNELS = {"popc": 1, "tc": 2, "tc_wm": 2, "tc_gather": 2, "tc_pull": 2, "tc_comp": 2, "tc_pull_gather": 2}
RING = {"tc": 1, "tc_wm": 2, "tc_gather": 2, "tc_pull": 3, "tc_comp": 1, "tc_pull_gather": 3}
OPERAND = {"tc": 1, "tc_comp": 2}


def make_sim(ranc, net, kernel, **kw):
    sim = ranc.Simulator(net, **kw)
    if kernel in RING:
        try:
            sim.set_option(ranc.OPT_KERNEL, KERNELS[kernel])
            sim.set_option(ranc.OPT_INPUT_DECODE, 0 if kernel in ("tc_gather", "tc_pull_gather") else 1)
            sim.set_option(ranc.OPT_RING_LAYOUT, RING[kernel])
            sim.set_option(ranc.OPT_OPERAND, OPERAND.get(kernel, 0))
        except ranc.RancError as e:
            sim.close()
            assert e.code == "RANC_E_CONFIG"
            pytest.skip("outside the tensor-core envelope")
    elif kernel:
        sim.set_option(ranc.OPT_KERNEL, KERNELS[kernel])
    return sim


@pytest.fixture(params=["popc", "tc", "tc_wm", "tc_gather", "tc_pull", "tc_comp"])
def kernel(request):
    return request.param


def per_tick(ranc, oracle_mod, net, inp, T, tile=None, kernel=None):
    sim = make_sim(ranc, net, kernel)
    if tile:
        sim.set_option(ranc.OPT_SAMPLE_TILE, tile)
    sim.set_trace(ranc.TRACE_SPIKE_RASTER | ranc.TRACE_OUTPUT_EVENTS)
    sim.load_inputs(inp)
    if kernel:
        assert sim.info()["kernel"] == KERNELS[kernel]
    if kernel in RING:
        assert sim.info()["ring_layout"] == RING[kernel]
    o = oracle_mod.Oracle(net, inp)
    for t in range(T):
        sim.run(1)
        o.run(1)
        if t == 0 and kernel in OPERAND:
            assert sim.info()["operand"] == OPERAND[kernel]
        where = f"{net.name} tick {t}"
        assert np.array_equal(sim.potentials(), o.potentials()), where + " potentials"
        assert np.array_equal(sim.raster()[0], o.fired()), where + " fired"
        assert np.array_equal(sim.pending(), o.pending()), where + " pending"
        assert np.array_equal(sim.outputs(), o.counts()), where + " counts"
    sim.close()
    return o


def final_state(ranc, oracle_mod, net, inp, T, tile=None, events=True, kernel=None):
    sim = make_sim(ranc, net, kernel)
    if tile:
        sim.set_option(ranc.OPT_SAMPLE_TILE, tile)
    if events:
        sim.set_trace(ranc.TRACE_OUTPUT_EVENTS)
    sim.load_inputs(inp).run(T)
    o = oracle_mod.Oracle(net, inp).run(T)
    assert np.array_equal(sim.outputs(), o.counts())
    assert np.array_equal(sim.potentials(), o.potentials())
    assert np.array_equal(sim.pending(), o.pending())
    if events:
        assert np.array_equal(sim.events(), o.events())
    sim.close()
    return o


def test_config1_every_tick(ranc, oracle_mod, kernel):
    net, inp = config1()
    o = per_tick(ranc, oracle_mod, net, inp, 64, kernel=kernel)
    assert o.counts().sum() > 0 and o.pending().sum() > 0


@pytest.mark.parametrize("seed", range(0, 200))
def test_tiny_every_tick(ranc, oracle_mod, seed, kernel):
    net, inp = tiny_case(seed)
    per_tick(ranc, oracle_mod, net, inp, 20, kernel=kernel)


@pytest.mark.parametrize("seed", range(0, 40))
def test_corpus_every_tick(ranc, oracle_mod, seed, kernel):
    net, inp = corpus_case(seed)
    per_tick(ranc, oracle_mod, net, inp, 12, kernel=kernel)


@pytest.mark.parametrize("seed", range(0, 40, 3))
def test_history_scheduler_gathered_inputs(ranc, oracle_mod, seed):
    """The history scheduler with per-tick input gathering (no load-time
    decode): input words transposed into the per-axon masks (a2)."""
    net, inp = corpus_case(seed)
    per_tick(ranc, oracle_mod, net, inp, 12, kernel="tc_pull_gather")


def test_history_scheduler_gathered_inputs_config2(ranc, oracle_mod):
    net, inp = config2(S=130)
    final_state(ranc, oracle_mod, net, inp, 17, kernel="tc_pull_gather")


@pytest.mark.parametrize("tile", [1, 3, 64])
def test_config2_full(ranc, oracle_mod, tile, kernel):
    net, inp = config2(S=300)
    o = final_state(ranc, oracle_mod, net, inp, 17, tile=tile, kernel=kernel)
    assert o.counts().sum() > 0


def test_config2_1000_samples(ranc, oracle_mod, kernel):
    net, inp = config2(S=1000)
    final_state(ranc, oracle_mod, net, inp, 17, kernel=kernel)


def test_config5_small_mesh(ranc, oracle_mod, kernel):
    net, inp = config5(S=5, T=40, grid=8)
    o = final_state(ranc, oracle_mod, net, inp, 40, kernel=kernel)
    assert o.pending().sum() > 0


def test_config5_global_every_tick(ranc, oracle_mod, kernel):
    net, inp = config5(S=3, T=20, grid=6, variant="global")
    per_tick(ranc, oracle_mod, net, inp, 20, kernel=kernel)


def test_config3_full_size_sampled(ranc, oracle_mod, kernel):
    """Config 3 at BASELINE size (10000 samples, 19 ticks, bench launch
    configuration) on the GPU; the oracle recomputes a spread of samples one
    by one (samples are independent, pinned by batch composition)."""
    net, inp = config3(S=10000)
    T = net.meta["T"]
    sim = make_sim(ranc, net, kernel)
    sim.load_inputs(inp).run(T)
    cnt = sim.outputs()
    pot = sim.potentials()
    pick = [0, 1, 2, 4097, 5000, 7777, 9998, 9999]
    o = oracle_mod.Oracle(net, inp.subset(pick)).run(T)
    assert np.array_equal(cnt[pick], o.counts())
    assert np.array_equal(pot[pick], o.potentials())
    assert cnt.sum() > 0
    sim.close()


@pytest.mark.parametrize("variant", ["vmm32", "vmm60", "vmm256"])
def test_vmm_closed_form_on_gpu(ranc, variant, kernel):
    """P6: the GPU's class counts equal M+ x and M- x (numpy), independent of
    the oracle."""
    from workloads.gen import VMM_VARIANTS
    net, inp = vmm(S=200, seed=1004, **VMM_VARIANTS[variant])
    M, X = net.meta["M"], net.meta["X"]
    sim = make_sim(ranc, net, kernel)
    sim.load_inputs(inp).run(net.meta["T"])
    cnt = sim.outputs()
    assert np.array_equal(cnt[:, 0::2], X @ np.maximum(M, 0).T)
    assert np.array_equal(cnt[:, 1::2], X @ np.maximum(-M, 0).T)
    sim.close()


def test_vmm_small_vs_oracle(ranc, oracle_mod, kernel):
    net, inp = vmm(16, 10, 7, 5, S=20, seed=5, block_in=8)
    final_state(ranc, oracle_mod, net, inp, net.meta["T"], kernel=kernel)


def test_resumable_and_reload(ranc, oracle_mod, kernel):
    net, inp = config1(T=40)
    sim = make_sim(ranc, net, kernel)
    sim.load_inputs(inp).run(7).run(0).run(33)
    p1, c1 = sim.potentials(), sim.outputs()
    sim.load_inputs(inp).run(40)
    assert np.array_equal(sim.potentials(), p1) and np.array_equal(sim.outputs(), c1)
    sim.reset().run(40)
    assert np.array_equal(sim.potentials(), p1) and np.array_equal(sim.outputs(), c1)
    o = oracle_mod.Oracle(net, inp).run(40)
    assert np.array_equal(p1, o.potentials())
    assert sim.now == 40
    sim.close()


def test_ticks_beyond_inputs_and_zero_ticks(ranc, oracle_mod, kernel):
    net, inp = config2(S=5)
    final_state(ranc, oracle_mod, net, inp, 30, kernel=kernel)
    sim = make_sim(ranc, net, kernel)
    sim.load_inputs(inp).run(0)
    assert np.array_equal(sim.potentials(), np.broadcast_to(net.initial_potential, (5, 5, 256)))
    sim.close()


def test_torch_stream_and_allocator(ranc, oracle_mod):
    import torch
    net, inp = config2(S=17)
    s = torch.cuda.Stream()
    sim = ranc.Simulator(net, stream=s, torch_allocator=True)
    sim.load_inputs(inp).run(17)
    o = oracle_mod.Oracle(net, inp).run(17)
    assert np.array_equal(sim.outputs(), o.counts())
    sim.close()


def test_call_order_errors(ranc):
    net, inp = config1(T=4)
    sim = ranc.Simulator(net)
    with pytest.raises(ranc.RancError) as ei:
        sim.run(1)
    assert ei.value.code == "RANC_E_STATE"
    sim.load_inputs(inp)
    with pytest.raises(ranc.RancError) as ei:
        sim._ck(sim.lib.ranc_read_outputs(sim.h, None, 3))
    assert ei.value.code == "RANC_E_SIZE"
    sim.close()


def test_kernel_switch_at_reset(ranc, oracle_mod):
    """The kernel variant is latched at reset; switching between runs gives
    the same results (the potential layout is re-initialised)."""
    net, inp = config2(S=70)
    sim = ranc.Simulator(net)
    assert sim.info()["kernel"] in (1, 2)
    res = []
    for k in (1, 2, 1):
        sim.set_option(ranc.OPT_KERNEL, k)
        sim.load_inputs(inp).run(9)
        assert sim.info()["kernel"] == k
        res.append((sim.potentials(), sim.outputs(), sim.pending()))
    for r in res[1:]:
        for a, b in zip(res[0], r):
            assert np.array_equal(a, b)
    o = oracle_mod.Oracle(net, inp).run(9)
    assert np.array_equal(res[0][0], o.potentials())
    sim.close()


def test_ring_layout_switch_at_reset(ranc, oracle_mod):
    """The ring layout is latched at reset (decoded inputs follow it); every
    layout gives the oracle's results, and the automatic choice is sample-major
    for the block-routed MNIST net and word-major for the random mesh."""
    net, inp = config2(S=70)
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_KERNEL, 2)
    o = oracle_mod.Oracle(net, inp).run(9)
    for lay, want in ((0, 1), (2, 2), (1, 1), (2, 2)):
        sim.set_option(ranc.OPT_RING_LAYOUT, lay)
        sim.load_inputs(inp).run(4)
        assert sim.info()["ring_layout"] == want
        sim.run(5)
        assert np.array_equal(sim.potentials(), o.potentials())
        assert np.array_equal(sim.outputs(), o.counts())
        assert np.array_equal(sim.pending(), o.pending())
    sim.close()
    with pytest.raises(ranc.RancError) as ei:
        s2 = ranc.Simulator(net)
        try:
            s2.set_option(ranc.OPT_RING_LAYOUT, 4)
        finally:
            s2.close()
    assert ei.value.code == "RANC_E_ARG"
    net5, inp5 = config5(S=64, T=4, grid=8)
    sim = ranc.Simulator(net5)
    sim.set_option(ranc.OPT_KERNEL, 2)
    sim.load_inputs(inp5)
    assert sim.info()["ring_layout"] == 2   # 64 items: the multi-tick launch keeps the ring
    sim.close()
    # more than two 64-sample tiles per SM: the history scheduler, and the
    # compact operand on its per-tick launches
    net5, inp5 = config5(S=64, T=4, grid=20)
    sim = ranc.Simulator(net5)
    sim.set_option(ranc.OPT_KERNEL, 2)
    sim.load_inputs(inp5).run(2)
    assert (sim.info()["ring_layout"], sim.info()["operand"]) == (3, 2)
    o = oracle_mod.Oracle(net5, inp5).run(2)
    assert np.array_equal(sim.potentials(), o.potentials())
    assert np.array_equal(sim.pending(), o.pending())
    sim.close()


def test_tc_envelope_rejects_wide_weights(ranc):
    """Weights of any valid width run on the tensor cores (-128..127: one s8
    operand; 16-bit: w = 256*hi + lo, a u8 and an s8 operand), and cores of up
    to 1024 neurons and axons (neuron groups, K chunks of 512 axons); 16-bit
    weights on 1024 axons do not fit the shared memory and are refused."""
    from workloads.gen import random_network
    net = random_network(3, 2, 1, 64, 64, 4, 3, wb=16)
    net.weight[0, 0, :2] = [-32768, 32767]
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_KERNEL, 2)   # 16-bit weights: accepted
    sim.close()
    net = random_network(3, 1, 1, 64, 300, 4, 3, wb=16)
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_KERNEL, 2)   # > 256 neurons: neuron groups
    sim.close()
    net = random_network(3, 1, 1, 600, 64, 4, 3, wb=8)
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_KERNEL, 2)   # > 512 axons: K chunks of 512
    sim.close()
    net = random_network(3, 1, 1, 1024, 64, 4, 3, wb=16)
    sim = ranc.Simulator(net)
    with pytest.raises(ranc.RancError) as ei:
        sim.set_option(ranc.OPT_KERNEL, 2)   # 1024 axons and 16-bit weights: beyond 227 KB, popcount only
    assert ei.value.code == "RANC_E_CONFIG"
    sim.close()


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("wk", ["tc", "tc_wm"])
def test_wide_weights_every_tick(ranc, oracle_mod, seed, wk):
    """Weights beyond int8 (wb 10..16, full range, incl. the extremes and
    multiples of 128 / 256) on the tensor-core path: w = 256*hi + lo, two MMAs, two
    TMEM accumulators; full state against the oracle every tick, 70 samples
    (a ragged second tile)."""
    from workloads.gen import bernoulli_inputs, random_network
    from workloads.rng import substream
    wb = [10, 12, 15, 16][seed]
    net = random_network(100 + seed, 3, 2, 256, 256, 4, 3, wb=wb, I=64)
    lo, hi = -(1 << (wb - 1)), (1 << (wb - 1)) - 1
    net.weight[0, :4, :] = [[lo, hi, -128, 128], [127, -127, 0, -129], [255, -256, 384, -385], [lo, lo, hi, hi]]
    inp = bernoulli_inputs(substream(200 + seed, "wide-inputs"), 70, 6, net.num_lines, 0.3)
    o = per_tick(ranc, oracle_mod, net, inp, 10, kernel=wk)
    assert o.counts().sum() > 0


# ---------------------------------------------------------------------------
# core-sharded mode, exercised through a loopback group on one GPU
# ---------------------------------------------------------------------------

def _core_sharded(ranc, net, inp, T, world, kernel):
    sims = []
    for r in range(world):
        sims.append(make_sim(ranc, net, kernel))
    ranc.Simulator.init_loopback(sims)
    for s in sims:
        s.set_trace(ranc.TRACE_OUTPUT_EVENTS)
        s.load_inputs(inp)
    ranc.Simulator.run_loopback(sims, T)
    return sims


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("variant", ["local", "global"])
def test_core_sharded_loopback_matches_oracle(ranc, oracle_mod, kernel, world, variant):
    net, inp = config5(S=4, T=30, grid=6, variant=variant)
    T = 30
    sims = _core_sharded(ranc, net, inp, T, world, kernel)
    o = oracle_mod.Oracle(net, inp).run(T)
    pot, pend = o.potentials(), o.pending()
    counts = np.zeros_like(o.counts())
    events = []
    for s in sims:
        i = s.info()
        lo, g = i["core_lo"], i["cores_local"]
        assert i["shard_mode"] == 1
        assert np.array_equal(s.potentials(), pot[:, lo:lo + g]), "potentials of the local band"
        assert np.array_equal(s.pending(), pend[:, lo:lo + g]), "pending of the local band"
        counts += s.outputs()
        events.append(s.events())
    assert np.array_equal(counts, o.counts())
    ev = np.concatenate(events)
    ev = ev[np.lexsort((ev[:, 4], ev[:, 2], ev[:, 3], ev[:, 1], ev[:, 0]))]
    assert np.array_equal(ev, o.events())
    assert sum(s.info()["exchange_bytes"] for s in sims) > 0
    for s in sims:
        s.close()


def test_core_sharded_random_corpus(ranc, oracle_mod, kernel):
    from workloads.gen import random_network, random_inputs
    for seed in range(6):
        net = random_network(seed, 3, 4, 40, 33, 3, 4, C=3, I=20)
        inp = random_inputs(seed, net, 3, 10, p=0.3)
        sims = _core_sharded(ranc, net, inp, 12, 2, kernel)
        o = oracle_mod.Oracle(net, inp).run(12)
        got = np.concatenate([s.potentials() for s in sims], axis=1)
        assert np.array_equal(got, o.potentials()), seed
        assert np.array_equal(sum(s.outputs() for s in sims), o.counts()), seed
        for s in sims:
            s.close()


def test_sample_sharded_comm_world1(ranc, oracle_mod):
    """NCCL communicator with one rank: gather == local outputs."""
    net, inp = config2(S=20)
    sim = ranc.Simulator(net)
    sim.comm_init(ranc.Simulator.unique_id(), 1, 0)
    sim.load_inputs(inp).run(17)
    assert np.array_equal(sim.gather_outputs(20, 0, 0), sim.outputs())
    sim.close()


# ---- streaming mode: one cooperative launch per run ----------


def stream_run(ranc, oracle_mod, net, inp, pieces, stream, trace=True):
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_KERNEL, 1)
    sim.set_option(ranc.OPT_STREAM, stream)
    if trace:
        sim.set_trace(ranc.TRACE_OUTPUT_EVENTS)
    sim.load_inputs(inp)
    assert sim.info()["kernel"] == 1
    launches0 = sim.info()["kernel_launches"]
    for k in pieces:
        sim.run(k)
    launches = sim.info()["kernel_launches"] - launches0
    T = sum(pieces)
    o = oracle_mod.Oracle(net, inp).run(T)
    assert np.array_equal(sim.outputs(), o.counts())
    assert np.array_equal(sim.potentials(), o.potentials())
    assert np.array_equal(sim.pending(), o.pending())
    if trace and len(pieces) == 1:   # the trace covers the last ranc_run_ticks call
        assert np.array_equal(sim.events(), o.events())
    sim.close()
    return launches


@pytest.mark.parametrize("stream", [1, 2])
def test_stream_config3_one_image_per_tick(ranc, oracle_mod, stream):
    net, inp = config3_stream(40)
    T = net.meta["T"]
    launches = stream_run(ranc, oracle_mod, net, inp, [T], stream)
    assert launches == (1 if stream == 2 else T)


def test_stream_resumable_in_pieces(ranc, oracle_mod):
    net, inp = config3_stream(30)
    stream_run(ranc, oracle_mod, net, inp, [1, 7, 2, 13, 11], 2)


@pytest.mark.parametrize("stream", [0, 2])
def test_stream_config1_and_config2(ranc, oracle_mod, stream):
    net, inp = config1(T=64)
    stream_run(ranc, oracle_mod, net, inp, [64], stream)
    net, inp = config2(S=48)
    stream_run(ranc, oracle_mod, net, inp, [5, net.meta["T"] - 5], stream)


@pytest.mark.parametrize("seed", range(0, 30))
def test_stream_corpus(ranc, oracle_mod, seed):
    net, inp = corpus_case(seed)
    stream_run(ranc, oracle_mod, net, inp, [3, 17], 2, trace=False)


def test_auto_kernel_small_batch_uses_popcount(ranc):
    net, inp = config3_stream(5)
    sim = ranc.Simulator(net)
    sim.load_inputs(inp)
    assert sim.info()["kernel"] == 1   # S = 1 <= 64: popcount path (+ streaming launch)
    sim.close()


def test_stream_multi_item_kernel(ranc, oracle_mod):
    # 512 cores x 2 samples (sample tile 1) = 1024 items: more than one item per
    # CTA, so the multi-item streaming kernel (resident potentials) runs
    net, inp = config3(S=2)
    stream_run(ranc, oracle_mod, net, inp, [net.meta["T"]], 2)
    stream_run(ranc, oracle_mod, net, inp, [4, 15], 2, trace=False)


# ---- design-space sweep batching ------------------------------


def test_sweep_tiled_variants_on_gpu(ranc, oracle_mod, kernel):
    from paper_2404_16208_b200.sweep import split_counts, split_potentials, tile_variants
    net, inp = config2(S=130)
    variants = sweep_variants(net, 5)
    tiled = tile_variants(variants)
    T = net.meta["T"]
    sim = make_sim(ranc, tiled, kernel)
    sim.load_inputs(inp).run(T)
    cnt = split_counts(sim.outputs(), 5, net.num_classes)
    pot = split_potentials(sim.potentials(), 5, net.G)
    sim.close()
    for v, vn in enumerate(variants):
        o = oracle_mod.Oracle(vn, inp).run(T)
        assert np.array_equal(cnt[:, v], o.counts()), f"variant {v}"
        assert np.array_equal(pot[:, v], o.potentials()), f"variant {v}"


# ---- tensor-core path: all ticks of a call in one cooperative launch -----------


@pytest.mark.parametrize("stream", [1, 0])
def test_tc_multi_tick_launch(ranc, oracle_mod, stream):
    net, inp = config2(S=130)
    T = net.meta["T"]
    for pieces in ([T], [1, 6, T - 7]):
        sim = ranc.Simulator(net)
        sim.set_option(ranc.OPT_KERNEL, 2)
        sim.set_option(ranc.OPT_STREAM, stream)
        sim.set_trace(ranc.TRACE_OUTPUT_EVENTS)
        sim.load_inputs(inp)
        l0 = sim.info()["kernel_launches"]
        for k in pieces:
            sim.run(k)
        launches = sim.info()["kernel_launches"] - l0
        o = oracle_mod.Oracle(net, inp).run(T)
        assert np.array_equal(sim.outputs(), o.counts())
        assert np.array_equal(sim.potentials(), o.potentials())
        assert np.array_equal(sim.pending(), o.pending())
        if len(pieces) == 1:
            assert np.array_equal(sim.events(), o.events())
            assert launches == (1 if stream == 0 else T)
        sim.close()


@pytest.mark.parametrize("S", [1650, 1600])
@pytest.mark.parametrize("ring", [1, 2])
def test_tc_multi_tick_two_items_per_cta(ranc, oracle_mod, S, ring):
    """More than 148 and at most 296 (core, tile) items: the multi-tick launch
    keeps two potential tiles per CTA in shared memory (6 random 128x128
    cores; S = 1650: 156 items, pairs of one core; S = 1600: 150 items, some
    CTAs straddle two cores, a ragged last tile), in one call and resumed in
    pieces."""
    from workloads.gen import bernoulli_inputs, random_network
    from workloads.rng import substream
    net = random_network(7, 3, 2, 128, 128, 4, 3, I=64, wb=8)
    net.weight[:] = np.maximum(net.weight, -127)   # int8 operand (the wide variant has no multi-tick launch)
    inp = bernoulli_inputs(substream(17, "two-items"), S, 6, net.num_lines, 0.3)
    T = 20
    o = oracle_mod.Oracle(net, inp).run(T)
    for pieces in ([T], [1, 6, T - 7]):
        sim = ranc.Simulator(net)
        sim.set_option(ranc.OPT_KERNEL, 2)
        sim.set_option(ranc.OPT_RING_LAYOUT, ring)
        sim.set_trace(ranc.TRACE_OUTPUT_EVENTS)
        sim.load_inputs(inp)
        l0 = sim.info()["kernel_launches"]
        for k in pieces:
            sim.run(k)
        assert sim.info()["kernel_launches"] - l0 == len(pieces)   # one cooperative launch per call
        assert np.array_equal(sim.outputs(), o.counts())
        assert np.array_equal(sim.potentials(), o.potentials())
        assert np.array_equal(sim.pending(), o.pending())
        if len(pieces) == 1:
            assert np.array_equal(sim.events(), o.events())
        sim.close()


def test_tc_multi_tick_corpus_and_vmm(ranc, oracle_mod):
    for seed in range(12):
        net, inp = corpus_case(seed)
        try:
            final_state(ranc, oracle_mod, net, inp, 20, kernel="tc")
        except pytest.skip.Exception:
            continue
    net, inp = config4("vmm32", S=20)
    final_state(ranc, oracle_mod, net, inp, net.meta["T"], kernel="tc", events=False)


# ---- state digest (RANC_TRACE_STATE_DIGEST) ---------------------


def digest_check(ranc, oracle_mod, net, inp, T, kernel):
    sim = make_sim(ranc, net, kernel)
    sim.set_trace(ranc.TRACE_STATE_DIGEST)
    sim.load_inputs(inp).run(T)
    got = sim.digests()
    sim.close()
    o = oracle_mod.Oracle(net, inp)
    for t in range(T):
        o.run(1)
        assert np.array_equal(got[t], o.digest()), f"{net.name} tick {t}"


def test_digest_config2_every_tick(ranc, oracle_mod, kernel):
    net, inp = config2(S=70)
    digest_check(ranc, oracle_mod, net, inp, net.meta["T"], kernel)


@pytest.mark.parametrize("seed", range(0, 10))
def test_digest_corpus(ranc, oracle_mod, seed, kernel):
    net, inp = corpus_case(seed)
    digest_check(ranc, oracle_mod, net, inp, 12, kernel)


def test_digest_config3_full_width(ranc, oracle_mod):
    # all 512 cores, a 3-sample slice checked against the oracle tick by tick
    net, inp = config3(S=3)
    digest_check(ranc, oracle_mod, net, inp, net.meta["T"], "tc")


def test_digest_core_sharded_shards_add_up(ranc, oracle_mod, kernel):
    # the digest is a sum over cores: the shards' digests add up (mod 2^64)
    # to the whole network's, tick by tick
    net, inp = config5(S=3, T=14, grid=6, variant="global")
    T = 14
    sims = [make_sim(ranc, net, kernel) for _ in range(3)]
    ranc.Simulator.init_loopback(sims)
    for s in sims:
        s.set_trace(ranc.TRACE_STATE_DIGEST)
        s.load_inputs(inp)
    ranc.Simulator.run_loopback(sims, T)
    total = sims[0].digests().copy()
    for s in sims[1:]:
        total += s.digests()   # uint64 wrap-around = mod 2^64
    for s in sims:
        s.close()
    o = oracle_mod.Oracle(net, inp)
    for t in range(T):
        o.run(1)
        assert np.array_equal(total[t], o.digest()), f"tick {t}"


# ---- mutation tests (a fault-injected parallel build must FAIL
# with a located divergence; RANC_OPT_DEBUG_FAULT) -------------------------------


@pytest.mark.parametrize("fault,variant", [(0, "tc_multi"), (1, "tc_multi"), (0, "popc_stream"), (1, "popc_stream"),
                                           (2, "tc"), (2, "popc")])
def test_fault_injection_is_caught(ranc, fault, variant):
    from verify import first_divergence, verdict
    if fault == 2:   # early delivery needs delays >= 2: the D = 15 random mesh
        net, inp = config5(S=40, T=20, grid=6)
    else:            # the missing barrier: the 5-core net's cross-core deposits
        net, inp = config2(S=130 if variant.startswith("tc") else 48)
    T = net.meta["T"]
    sim = ranc.Simulator(net)
    sim.set_option(ranc.OPT_KERNEL, 2 if variant.startswith("tc") else 1)
    sim.set_option(ranc.OPT_STREAM, 2 if variant.endswith(("multi", "stream")) else 1)
    sim.set_option(ranc.OPT_DEBUG_FAULT, fault)
    sim.set_trace(ranc.TRACE_SPIKE_RASTER)
    sim.load_inputs(inp)
    l0 = sim.info()["kernel_launches"]
    div = first_divergence(sim, net, inp, T)
    launches = sim.info()["kernel_launches"] - l0
    sim.close()
    if variant.endswith(("multi", "stream")):
        assert launches == 1, "the barrier fault needs the one-launch (grid barrier) path"
    msg = verdict(div)
    if fault == 0:
        assert div is None, msg
    else:
        assert div is not None, f"fault {fault} on {variant} was NOT detected"
        assert msg.startswith("FAIL: first divergence at tick") and div["tick"] >= 1, msg
        print(msg)
