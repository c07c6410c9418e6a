"""Hand-built tiny networks for the closed-form pins."""
from __future__ import annotations

import numpy as np

from workloads.gen import _blank
from workloads.netdef import KIND_OUTPUT, KIND_ROUTE, MODE_ABS, MODE_LIN, Inputs, Network


def single_neuron(w=1, leak=0, pos=1, neg=-(1 << 15), reset=0, mode=MODE_ABS, pb=16,
                  init=0, wb=16, lb=16, tb=16, rb=16, D=1):
    """1x1 grid, A = N = 1, axon 0 fed by input line 0, neuron -> output class 0."""
    net = _blank(1, 1, 1, 1, 1, D, 1, 1, pb=pb, wb=wb, lb=lb, tb=tb, rb=rb, name="single")
    net.input_line[0, 0] = 0
    net.crossbar[0, 0, 0] = 1
    net.weight[0, 0, 0] = w
    net.leak[0, 0] = leak
    net.pos_threshold[0, 0] = pos
    net.neg_threshold[0, 0] = neg
    net.reset_potential[0, 0] = reset
    net.reset_mode[0, 0] = mode
    net.initial_potential[0, 0] = init
    net.dest_kind[0, 0] = KIND_OUTPUT
    net.out_class[0, 0] = 0
    return net


def input_every_tick(T, S=1):
    return Inputs.from_dense(np.ones((S, T, 1), bool))


def input_at(ticks, T, I=1, line=0, S=1):
    spk = np.zeros((S, T, I), bool)
    for t in ticks:
        spk[:, t, line] = True
    return Inputs.from_dense(spk)


def no_input(S=1, T=1, I=1):
    return Inputs.from_dense(np.zeros((S, T, I), bool))


def relay_chain(L, d, D=None):
    """L cores in a row, one axon/neuron each, theta+ = 1, w = 1; core i routes
    to core i+1 axon 0 with delay d; the last core is on the output bus."""
    D = D or d
    net = _blank(L, 1, 1, 1, 1, D, 1, 1, name="relay")
    net.crossbar[:, 0, 0] = 1
    net.weight[:, 0, 0] = 1
    net.pos_threshold[:] = 1
    net.neg_threshold[:] = -(1 << 15)
    net.input_line[0, 0] = 0
    for c in range(L - 1):
        net.dest_kind[c, 0] = KIND_ROUTE
        net.dest_dx[c, 0] = 1
        net.dest_axon[c, 0] = 0
        net.dest_delay[c, 0] = d
    net.dest_kind[L - 1, 0] = KIND_OUTPUT
    return net


def permute_axons(net: Network, perms):
    """Relabel the axons of every core c by perms[c] (new index = perms[c][old]),
    rewriting crossbar, types, input lines and every route that targets c."""
    out = net.copy()
    conn = net.conn_dense()
    newconn = np.zeros_like(conn)
    for c in range(net.G):
        p = perms[c]
        newconn[c][:, p] = conn[c]
        out.axon_type[c][p] = net.axon_type[c]
        out.input_line[c][p] = net.input_line[c]
    out.crossbar[:] = Network.pack_conn(newconn)
    xs = np.arange(net.G) % net.grid_w
    ys = np.arange(net.G) // net.grid_w
    for c in range(net.G):
        for n in range(net.neurons):
            if net.dest_kind[c, n] == KIND_ROUTE:
                dc = (ys[c] + net.dest_dy[c, n]) * net.grid_w + xs[c] + net.dest_dx[c, n]
                out.dest_axon[c, n] = perms[dc][net.dest_axon[c, n]]
    return out


def permute_neurons(net: Network, perms):
    """Relabel neurons of core c: new index = perms[c][old]."""
    out = net.copy()
    for name in ("weight", "leak", "pos_threshold", "neg_threshold", "reset_potential",
                 "initial_potential", "reset_mode", "dest_kind", "dest_dx", "dest_dy",
                 "dest_axon", "dest_delay", "out_class", "crossbar"):
        src = getattr(net, name)
        dst = getattr(out, name)
        for c in range(net.G):
            dst[c][perms[c]] = src[c]
    return out
