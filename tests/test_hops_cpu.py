"""Hop-by-hop routing check (G18): the paper's router forwards
a packet one core per hop, x first, then y; the direct routing the
library implements must reach the same destination core.  A plain hop-by-hop
walk over random routes of the config-5 mesh (both variants) lands exactly on
(x + dx, y + dy) after |dx| + |dy| hops, never leaving the grid."""
import numpy as np
import pytest

from workloads.gen import config5


def hop_walk(x, y, dx, dy, W, H):
    hops = 0
    while dx != 0:
        s = 1 if dx > 0 else -1
        x += s
        dx -= s
        hops += 1
        assert 0 <= x < W
    while dy != 0:
        s = 1 if dy > 0 else -1
        y += s
        dy -= s
        hops += 1
        assert 0 <= y < H
    return x, y, hops


@pytest.mark.parametrize("variant", ["local", "global"])
def test_hop_by_hop_equals_direct(variant):
    net, _ = config5(S=1, T=1, grid=16, variant=variant)
    W = H = 16
    rng = np.random.default_rng(0)
    cores = rng.integers(0, net.G, 200)
    neurons = rng.integers(0, net.neurons, 200)
    checked = 0
    for c, n in zip(cores, neurons):
        if net.dest_kind[c, n] != 1:
            continue
        x, y = c % W, c // W
        dx, dy = int(net.dest_dx[c, n]), int(net.dest_dy[c, n])
        hx, hy, hops = hop_walk(x, y, dx, dy, W, H)
        assert (hx, hy) == (x + dx, y + dy)
        assert hops == abs(dx) + abs(dy)
        checked += 1
    assert checked > 100
