"""Core-sharded config 5 on ONE GPU as a loopback group: the
per-tick cost of W row bands with the exchange (pack -> copies -> unpack)
between them, against the unsharded run.  Prints one JSON line per world.

  python tools/loopback_bench.py [T] [world ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_16208_b200 as r  # noqa: E402
from workloads.gen import config5  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 100
worlds = [int(w) for w in sys.argv[2:]] or [1, 2, 4, 8]
for variant in ("local", "global"):
    net, inp = config5(S=64, T=T, variant=variant)
    for world in worlds:
        sims = [r.Simulator(net) for _ in range(world)]
        if world > 1:
            r.Simulator.init_loopback(sims)
        for s in sims:
            s.load_inputs(inp)
        run = (lambda k: r.Simulator.run_loopback(sims, k)) if world > 1 else (lambda k: sims[0].run(k).outputs())
        run(10)   # warm-up
        for s in sims:
            s.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run(T)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ex = sum(s.info()["exchange_bytes"] for s in sims)
        print(json.dumps({"workload": net.name, "world": world, "ticks": T, "ms_per_tick": dt / T * 1e3,
                          "exchange_bytes_per_tick": ex, "cores_per_shard": sims[0].info()["cores_local"],
                          "note": "loopback group on one GPU: all shards share the device, so ms_per_tick is the "
                                  "serialised cost of every shard plus the exchange"}), flush=True)
        for s in sims:
            s.close()
