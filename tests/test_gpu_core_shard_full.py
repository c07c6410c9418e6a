"""Core-sharded mode at the benchmarked size: config 5's 64x64
mesh split into 8 row bands (512 cores per shard, the 8-GPU layout), run as a
loopback group on one GPU (the same pack / exchange / unpack kernels as the
NCCL path, device copies instead of ncclSend/ncclRecv).  The shards' state
digests (G21) add up, tick by tick, to the oracle's for a sample slice and to
the single-context run's for every sample."""
import numpy as np
import pytest

from oracle_pool import oracle_digests
from workloads.gen import config5

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ranc():
    from paper_2404_16208_b200 import build
    build.build()
    import paper_2404_16208_b200 as m
    return m


@pytest.mark.parametrize("variant", ["local", "global"])
def test_config5_eight_shards_every_tick(ranc, variant):
    T, S, world = 40, 64, 8
    net, inp = config5(S=S, T=T, variant=variant)
    sims = [ranc.Simulator(net) for _ in range(world)]
    ranc.Simulator.init_loopback(sims)
    for s in sims:
        s.set_trace(ranc.TRACE_STATE_DIGEST)
        s.load_inputs(inp)
    ranc.Simulator.run_loopback(sims, T)
    total = sims[0].digests().copy()
    for s in sims[1:]:
        total += s.digests()   # uint64 wrap-around = mod 2^64
    bands = [(s.info()["core_lo"], s.info()["cores_local"]) for s in sims]
    assert [g for _, g in bands] == [512] * world and sum(s.info()["exchange_bytes"] for s in sims) > 0
    counts = sum(s.outputs().astype(np.int64) for s in sims)
    for s in sims:
        s.close()
    one = ranc.Simulator(net)
    one.set_trace(ranc.TRACE_STATE_DIGEST)
    one.load_inputs(inp).run(T)
    d1, c1 = one.digests(), one.outputs()
    one.close()
    assert np.array_equal(total, d1), "shard digests do not add up to the single-context run"
    assert np.array_equal(counts, c1)
    idx = np.array([0, 63])
    (ref, ref_c, _), = oracle_digests([(net, inp, idx, T)])
    for t in range(T):
        assert np.array_equal(total[t, idx], ref[t]), f"tick {t}"
    assert np.array_equal(counts[idx], ref_c)
