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
