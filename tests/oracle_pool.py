"""Fan the serial oracle out over the host cores (samples are independent
simulations, G14 / P9 batch composition), for parity checks at the
benchmarked sizes.  Test infrastructure: imports oracle/."""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_JOB = {}


def _digest_worker(args):
    idx, T = args
    from oracle.pyoracle import Oracle
    net, inp = _JOB["net"], _JOB["inp"]
    o = Oracle(net, inp.subset(idx))
    dig = np.zeros((T, len(idx)), np.uint64)
    for t in range(T):
        o.run(1)
        dig[t] = o.digest()
    return idx, dig, o.counts(), o.potentials()


def host_procs(cap=32):
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 1
    return max(1, min(n, cap))


def oracle_digests(jobs, procs=None):
    """jobs: list of (net, inputs, sample indices, T).  Returns, per job,
    (digests uint64 [T][len(idx)], counts [len(idx)][C], potentials
    [len(idx)][G][N]) of the oracle, one worker process per sample."""
    from oracle import pyoracle
    pyoracle.build()
    procs = procs or host_procs()
    out = []
    ctx = mp.get_context("fork")
    for net, inp, idx, T in jobs:
        _JOB["net"], _JOB["inp"] = net, inp
        idx = [int(i) for i in idx]
        with ctx.Pool(min(procs, len(idx))) as pool:
            parts = pool.map(_digest_worker, [([i], T) for i in idx])
        dig = np.concatenate([p[1] for p in parts], axis=1)
        cnt = np.concatenate([p[2] for p in parts], axis=0)
        pot = np.concatenate([p[3] for p in parts], axis=0)
        out.append((dig, cnt, pot))
    return out
