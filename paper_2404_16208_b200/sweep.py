"""Design-space sweep batching.

The paper's motivation for a fast simulator is sweeping architectural
parameters -- weights, leaks, thresholds, reset modes, bitwidths -- over the
same application.  Here V variants of one network are run in
ONE launch as an extra batch axis, with no kernel change: the variants are
stacked as disjoint blocks of rows of one larger core grid.

* variant v, core (x, y)  ->  core (x, v*H + y), i.e. core index v*G + c;
* routes are relative (dx, dy) and valid routes stay inside their own H rows,
  so the blocks never exchange spikes (Alg. 1 l.15-20 applied per block);
* input lines are shared: every variant sees the same input stream;
* output class k of variant v becomes class v*C + k, so
  ``counts.reshape(S, V, C)[:, v]`` are variant v's counts.

Cores are independent except through routes, so the tiled network computes,
block by block, exactly what each variant computes alone (pinned by
tests/test_sweep_cpu.py with the oracle).  This is host-side table building
(argument marshalling); the simulation itself runs in libranc.so.

Restrictions: the variants share A, N, the grid shape, C, I and the potential
bitwidth (pb decides saturation, G3); the other bitwidths are validation
limits only and take the maximum; K and D take the maximum (weights of the
extra types are zero).
"""
from __future__ import annotations

import dataclasses
from types import SimpleNamespace

import numpy as np

_PER_CORE = ["axon_type", "input_line", "crossbar", "weight", "leak", "pos_threshold", "neg_threshold",
             "reset_potential", "initial_potential", "reset_mode", "dest_kind", "dest_dx", "dest_dy",
             "dest_axon", "dest_delay", "out_class"]
_SAME = ["grid_w", "grid_h", "axons", "neurons", "num_classes", "num_lines", "potential_bits"]
_MAX = ["num_types", "max_delay", "weight_bits", "leak_bits", "threshold_bits", "reset_bits"]
KIND_OUTPUT = 2


def tile_variants(nets):
    """Stack V network variants into one network (see module docstring).
    Returns a network of the same type as nets[0] (a dataclass is rebuilt with
    dataclasses.replace, anything else becomes a SimpleNamespace)."""
    nets = list(nets)
    if not nets:
        raise ValueError("tile_variants: no variants")
    n0 = nets[0]
    for k in _SAME:
        vals = {int(getattr(n, k)) for n in nets}
        if len(vals) != 1:
            raise ValueError(f"tile_variants: variants differ in {k} ({sorted(vals)}); only parameters, "
                             "crossbars, weights, routes and the non-potential bitwidths may vary")
    V = len(nets)
    H = int(n0.grid_h)
    C = int(n0.num_classes)
    K = max(int(n.num_types) for n in nets)
    out = {k: max(int(getattr(n, k)) for n in nets) for k in _MAX}
    arrays = {}
    for name in _PER_CORE:
        parts = []
        for v, n in enumerate(nets):
            a = np.asarray(getattr(n, name))
            if name == "weight" and a.shape[-1] < K:
                a = np.concatenate([a, np.zeros(a.shape[:-1] + (K - a.shape[-1],), a.dtype)], axis=-1)
            if name == "out_class":
                kind = np.asarray(n.dest_kind)
                a = np.where(kind == KIND_OUTPUT, a.astype(np.int64) + v * C, a).astype(np.asarray(n.out_class).dtype)
            parts.append(a)
        arrays[name] = np.ascontiguousarray(np.concatenate(parts, axis=0))
    fields = dict(arrays, **out, grid_h=V * H, num_classes=V * C)
    if dataclasses.is_dataclass(n0):
        tiled = dataclasses.replace(n0, **fields)
    else:
        base = {k: getattr(n0, k) for k in _SAME}
        tiled = SimpleNamespace(**dict(base, **fields))
    meta = dict(getattr(n0, "meta", {}) or {})
    Ts = [n.meta.get("T") for n in nets if getattr(n, "meta", None) and n.meta.get("T") is not None]
    if Ts:
        meta["T"] = max(Ts)
    meta.update(variants=V, variant_rows=H, variant_classes=C)
    try:
        tiled.meta = meta
        tiled.name = f"{getattr(n0, 'name', 'net')}-sweep{V}"
    except AttributeError:
        pass
    return tiled


def split_counts(counts, V: int, C: int):
    """[S][V*C] class counts of a tiled run -> [S][V][C]."""
    counts = np.asarray(counts)
    return counts.reshape(counts.shape[0], V, C)


def split_potentials(pot, V: int, G: int):
    """[S][V*G][N] potentials of a tiled run -> [S][V][G][N]."""
    pot = np.asarray(pot)
    return pot.reshape(pot.shape[0], V, G, pot.shape[-1])
