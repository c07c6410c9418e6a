"""World-size-2 gloo tests of the sample-sharded multi-GPU logic on CPU
(SURVEY 4 T8): shard arithmetic, rank-order concatenation of the gathered
class counts, and shard invariance of the results (samples are independent
simulations, G14).  The per-shard simulation here is the oracle, so the test
runs without a GPU; the GPU path uses the same shard_range and root order."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_16208_b200.dist import shard_range


def test_shard_range_partitions():
    for S in (0, 1, 2, 7, 10, 999, 10000):
        for world in (1, 2, 3, 4, 8):
            got = [shard_range(S, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == S
            for (a, b), (c, d) in zip(got, got[1:]):
                assert b == c
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from workloads.gen import config2
        net, inp = config2(S=9)
        lo, hi = shard_range(inp.num_samples, world, rank)
        o = Oracle(net, inp.slice(lo, hi)).run(net.meta["T"])
        parts = [None] * world if rank == 0 else None
        dist.gather_object((rank, o.counts(), o.potentials()), parts, dst=0)
        if rank == 0:
            counts = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])])
            pots = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
            np.save(out + "_counts.npy", counts)
            np.save(out + "_pots.npy", pots)
    finally:
        dist.destroy_process_group()


def test_sample_sharded_gather_world2(tmp_path, oracle_mod):
    from workloads.gen import config2
    out = str(tmp_path / "r")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    net, inp = config2(S=9)
    full = oracle_mod.Oracle(net, inp).run(net.meta["T"])
    assert np.array_equal(np.load(out + "_counts.npy"), full.counts())
    assert np.array_equal(np.load(out + "_pots.npy"), full.potentials())


# ---- core-sharded plan of the product (ranc_plan_core_shards, host only) ----


def _route_model(net, world):
    """Python model of the row-band partition and of which cores must export
    their fired bits to which rank (SURVEY 8(e) core-sharded mode): core
    (x, y) belongs to rank r iff r*H//world <= y < (r+1)*H//world; a core
    sends to rank p != owner iff one of its ROUTE neurons targets a core of
    p's band (Alg. 1 l.15-20)."""
    H, Wg = net.grid_h, net.grid_w
    owner = np.zeros(net.G, int)
    for r in range(world):
        for y in range(r * H // world, (r + 1) * H // world):
            owner[y * Wg:(y + 1) * Wg] = r
    to = [set() for _ in range(world)]   # to[p] = global source cores routing into p's band
    for g in range(net.G):
        x, y = g % Wg, g // Wg
        for n in range(net.neurons):
            if net.dest_kind[g, n] != 1:
                continue
            d = (y + net.dest_dy[g, n]) * Wg + (x + net.dest_dx[g, n])
            if owner[d] != owner[g]:
                to[owner[d]].add(g)
    return owner, to


def _plan_worker(rank, world, port, out, variant):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_16208_b200 import Simulator
        from workloads.gen import config5
        net, _ = config5(S=1, T=1, grid=12, variant=variant)
        plan = Simulator.plan_core_shards(net, world, rank)
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        if rank == 0:
            import pickle
            with open(out, "wb") as f:
                pickle.dump(plans, f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,variant", [(2, "local"), (3, "global")])
def test_core_shard_plan_matches_route_model(tmp_path, world, variant):
    """Each rank plans its own band in its own process (gloo); the plans are
    gathered and checked against the Python route model and against each
    other: what rank r sends to p is exactly what p expects from r."""
    import pickle
    from workloads.gen import config5
    out = str(tmp_path / "plans.pkl")
    mp.spawn(_plan_worker, args=(world, _free_port(), out, variant), nprocs=world, join=True)
    plans = pickle.load(open(out, "rb"))
    net, _ = config5(S=1, T=1, grid=12, variant=variant)
    owner, to = _route_model(net, world)
    covered = 0
    for r, pl in enumerate(plans):
        mine = np.flatnonzero(owner == r)
        assert pl["core_lo"] == mine[0] and pl["cores_local"] == len(mine)
        covered += pl["cores_local"]
        for p in range(world):
            send_global = [pl["core_lo"] + c for c in pl["send"][p]]
            if p == r:
                assert send_global == [] and pl["recv"][p] == []
                continue
            assert send_global == sorted(g for g in to[p] if owner[g] == r), (r, p)
            assert pl["recv"][p] == sorted(g for g in to[r] if owner[g] == p), (r, p)
            # the two ends of every link agree
            assert send_global == plans[p]["recv"][r]
    assert covered == net.G
    assert any(pl["send"][p] for pl in plans for p in range(world))


def test_core_shard_plan_errors():
    from paper_2404_16208_b200 import RancError, Simulator
    from workloads.gen import config5
    net, _ = config5(S=1, T=1, grid=6)
    with pytest.raises(RancError) as ei:
        Simulator.plan_core_shards(net, 7, 0)   # more ranks than grid rows
    assert ei.value.code == "RANC_E_CONFIG" and "grid_h=6" in str(ei.value)
    n = int(np.flatnonzero(net.dest_kind[0] == 1)[0])
    net.dest_delay[0, n] = 0
    with pytest.raises(RancError) as ei:
        Simulator.plan_core_shards(net, 2, 0)   # validation runs first: a located error
    assert ei.value.code == "RANC_E_RANGE" and f"core (0,0) neuron {n}" in str(ei.value)


def test_sample_shards_match_gather_contract():
    """ranc_gather_outputs (include/ranc.h) derives every shard from
    S_total = n / C: rank r owns [r*b + min(r, m), ...), b = S_total // world,
    m = S_total % world; the binding's shard_range must produce exactly those
    (the C side rejects any other first_sample / size with RANC_E_SIZE)."""
    for S in (1, 5, 64, 999, 10000):
        for world in (1, 2, 3, 4, 8):
            b, m = divmod(S, world)
            for r in range(world):
                lo = r * b + min(r, m)
                hi = (r + 1) * b + min(r + 1, m)
                assert shard_range(S, world, r) == (lo, hi)
