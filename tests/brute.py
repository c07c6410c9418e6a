"""Independent dense NumPy brute force of the RANC tick.

Written separately from oracle/oracle.c so that a shared bug is unlikely:
  * pending spikes are indexed by ABSOLUTE tick (an array of T+D+1 rows),
    not by a ring buffer -- so it cannot share the ring's index arithmetic;
  * integration is one int64 matrix product per core,
    acc = spikes @ Weff with Weff[a, n] = conn[n, a] * w[n, type[a]]
    ("accumulate neuron potential"; the library routine np.matmul
    is the pin of step a3);
  * leak / thresholds / reset are vectorised with np.where;
  * routing marks pending[t + delay][dest core][dest axon].
Returns the full state after every tick for comparison with the oracle.
"""
from __future__ import annotations

import numpy as np


def run(net, inputs, T):
    G, A, N, K, D = net.G, net.axons, net.neurons, net.num_types, net.max_delay
    S = inputs.num_samples
    conn = net.conn_dense()                                   # [G][N][A]
    w = net.weight.astype(np.int64)                           # [G][N][K]
    typ = net.axon_type.astype(np.int64)                      # [G][A]
    # Weff[c][a][n] = conn[c][n][a] * w[c][n][type[c][a]]
    wsel = np.take_along_axis(w, np.broadcast_to(typ[:, None, :], (G, N, A)), axis=2)  # [G][N][A]
    Weff = np.transpose(conn * wsel, (0, 2, 1)).astype(np.int64)                       # [G][A][N]
    lines = inputs.dense(net.num_lines)                       # [S][T_in][I]
    lo = -(1 << (net.potential_bits - 1))
    hi = (1 << (net.potential_bits - 1)) - 1
    pot = np.broadcast_to(net.initial_potential.astype(np.int64), (S, G, N)).copy()
    pend = np.zeros((S, T + D + 1, G, A), bool)
    counts = np.zeros((S, net.num_classes), np.int64)
    events = []
    xs = np.arange(G) % net.grid_w
    ys = np.arange(G) // net.grid_w
    leak = net.leak.astype(np.int64)
    pth = net.pos_threshold.astype(np.int64)
    nth = net.neg_threshold.astype(np.int64)
    rst = net.reset_potential.astype(np.int64)
    lin = net.reset_mode.astype(bool)
    states = []
    for t in range(T):
        if t < inputs.num_input_ticks and net.num_lines > 0:
            il = net.input_line
            has = il >= 0
            for s in range(S):
                arr = np.zeros((G, A), bool)
                arr[has] = lines[s, t, il[has]]
                pend[s, t] |= arr
        spk = pend[:, t].astype(np.int64)                     # [S][G][A]
        acc = np.einsum("sga,gan->sgn", spk, Weff)            # int64 matmul per core
        v = pot + acc + leak
        fire = v >= pth
        neg = (~fire) & (v < nth)
        nv = np.where(fire, np.where(lin, v - pth, rst), np.where(neg, np.where(lin, v - nth, -rst), v))
        pot = np.clip(nv, lo, hi)
        for s, c, n in zip(*np.nonzero(fire)):
            kind = net.dest_kind[c, n]
            if kind == 1:
                dc = (ys[c] + net.dest_dy[c, n]) * net.grid_w + (xs[c] + net.dest_dx[c, n])
                pend[s, t + net.dest_delay[c, n], dc, net.dest_axon[c, n]] = True
            elif kind == 2:
                counts[s, net.out_class[c, n]] += 1
                events.append((s, t, xs[c], ys[c], n))
        pending = np.stack([pend[:, t + 1 + j] for j in range(D)], axis=2)  # [S][G][D][A]
        states.append(dict(pot=pot.copy(), fired=fire.copy(), pending=pending.copy(),
                           counts=counts.copy()))
    # canonical order (sample, tick, y, x, neuron)
    ev = np.array(sorted(events, key=lambda e: (e[0], e[1], e[3], e[2], e[4])),
                  np.int64).reshape(-1, 5)
    return states, ev
