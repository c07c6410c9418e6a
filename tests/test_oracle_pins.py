"""Pins of the oracle to things other than itself (
DESIGN.md section 4).  CPU only.

Every expected value below is either a SPEC/paper worked example (cited) or a
closed form derived from the mathematics of the neuron model, not a re-run of
the oracle's own loop.
"""
import math

import numpy as np
import pytest

from nets import input_at, input_every_tick, no_input, relay_chain, single_neuron
from workloads.netdef import MODE_ABS, MODE_LIN

NEG_OFF = -(1 << 15)


# --------------------------------------------------------------------------
# SPEC worked examples (P8)
# --------------------------------------------------------------------------

def test_spec_saturate_examples(oracle_mod):
    # S:65-67
    assert oracle_mod.saturate(5, 8) == 5
    assert oracle_mod.saturate(200, 8) == 127
    assert oracle_mod.saturate(-300, 8) == -128
    # idempotence
    for v in (-1000, -129, -128, 0, 127, 128, 4000):
        for b in (2, 4, 8, 16):
            s = oracle_mod.saturate(v, b)
            assert oracle_mod.saturate(s, b) == s
            assert -(1 << (b - 1)) <= s <= (1 << (b - 1)) - 1


def test_spec_integrate_examples(oracle_mod):
    # S:75-77
    assert oracle_mod.integrate(0, [0, 0], [1, 1], [0, 1], [2, -1, 0, 0]) == 0
    assert oracle_mod.integrate(0, [1, 1], [1, 1], [0, 1], [2, -1, 0, 0]) == 1
    assert oracle_mod.integrate(3, [1, 1], [1, 0], [0, 1], [2, -1, 0, 0]) == 5


def test_integrate_is_linear_and_permutation_invariant(oracle_mod):
    # linearity in disjoint spike sets, axon-order invariance,
    # all-zero connections give the base potential.  Pinned against np.dot.
    rng = np.random.default_rng(0)
    for _ in range(200):
        A = int(rng.integers(1, 40))
        sp = rng.integers(0, 2, A)
        cn = rng.integers(0, 2, A)
        ty = rng.integers(0, 4, A)
        w = rng.integers(-300, 300, 4)
        pot = int(rng.integers(-100, 100))
        want = pot + int(np.dot(sp * cn, w[ty]))
        assert oracle_mod.integrate(pot, sp, cn, ty, w) == want
        p = rng.permutation(A)
        assert oracle_mod.integrate(pot, sp[p], cn[p], ty[p], w) == want
        assert oracle_mod.integrate(pot, sp, np.zeros(A), ty, w) == pot


def test_spec_lif_examples(oracle_mod):
    # S:85-87 (single threshold; the negative threshold is put out of reach)
    assert oracle_mod.lif(0, 0, 1, NEG_OFF, 0, MODE_ABS, 8) == (0, False)
    assert oracle_mod.lif(5, -2, 3, NEG_OFF, 0, MODE_ABS, 8) == (0, True)
    assert oracle_mod.lif(2, 0, 3, NEG_OFF, 0, MODE_ABS, 8) == (2, False)


def test_lif_branches(oracle_mod):
    # G1: equality fires; G4: negative branch both modes; G3: compare unclamped v
    assert oracle_mod.lif(10, 0, 10, -5, 3, MODE_ABS, 16) == (3, True)
    assert oracle_mod.lif(10, 2, 10, -5, 3, MODE_LIN, 16) == (2, True)
    assert oracle_mod.lif(-6, 0, 10, -5, 3, MODE_ABS, 16) == (-3, False)
    assert oracle_mod.lif(-6, -1, 10, -5, 3, MODE_LIN, 16) == (-2, False)
    assert oracle_mod.lif(-5, 0, 10, -5, 3, MODE_ABS, 16) == (-5, False)   # not < -5
    # unclamped v = 300 >= 200 fires even though pb = 8 would clamp it to 127
    assert oracle_mod.lif(300, 0, 200, NEG_OFF, 0, MODE_ABS, 8) == (0, True)
    # the stored value is clamped
    assert oracle_mod.lif(150, 0, 200, NEG_OFF, 0, MODE_ABS, 8) == (127, False)
    assert oracle_mod.lif(-150, 0, 200, -1000, 0, MODE_ABS, 8) == (-128, False)


# --------------------------------------------------------------------------
# single-neuron closed forms (P2, P3, P5)
# --------------------------------------------------------------------------

def fired_trace(oracle_mod, net, inp, T):
    o = oracle_mod.Oracle(net, inp)
    fired, pots = [], []
    for _ in range(T):
        o.run(1)
        fired.append(int(o.fired()[0, 0, 0]))
        pots.append(int(o.potentials()[0, 0, 0]))
    return np.array(fired), np.array(pots), o


@pytest.mark.parametrize("w,lam,th", [(1, 0, 1), (1, 0, 5), (3, 1, 10), (7, -2, 13),
                                      (5, 0, 5), (2, 3, 25), (9, -1, 8)])
def test_abs_reset_period(oracle_mod, w, lam, th):
    # ABS reset to 0 with constant drive w+lam>0 fires every k = ceil(th/(w+lam))
    # ticks, first at tick k-1 (fires at equality, G1).
    T = 60
    net = single_neuron(w=w, leak=lam, pos=th, mode=MODE_ABS)
    f, _, o = fired_trace(oracle_mod, net, input_every_tick(T), T)
    k = math.ceil(th / (w + lam))
    want = np.array([(t + 1) % k == 0 for t in range(T)], int)
    assert np.array_equal(f, want)
    assert o.counts()[0, 0] == T // k
    ev = o.events()
    assert list(ev[:, 1]) == [t for t in range(T) if (t + 1) % k == 0]


@pytest.mark.parametrize("w,lam,th", [(1, 0, 1), (1, 0, 5), (3, 1, 10), (7, -2, 13),
                                      (4, 0, 6), (2, 3, 25), (5, 0, 5)])
def test_linear_reset_count(oracle_mod, w, lam, th):
    # LIN reset (v - th): cumulative spikes by tick t = floor((t+1)(w+lam)/th)
    # for 0 < w+lam <= th; potential = (t+1)(w+lam) mod th.
    T = 60
    r = w + lam
    net = single_neuron(w=w, leak=lam, pos=th, mode=MODE_LIN)
    f, p, _ = fired_trace(oracle_mod, net, input_every_tick(T), T)
    cum = np.cumsum(f)
    for t in range(T):
        assert cum[t] == ((t + 1) * r) // th
        assert p[t] == ((t + 1) * r) % th


@pytest.mark.parametrize("lam,th", [(1, 5), (3, 10), (4, 4), (7, 100)])
def test_leak_only_first_fire(oracle_mod, lam, th):
    # G2: leak is applied every tick even with no input: first spike at tick
    # ceil(th/lam) - 1.
    T = 120
    net = single_neuron(w=0, leak=lam, pos=th, mode=MODE_ABS)
    f, _, _ = fired_trace(oracle_mod, net, no_input(T=1), T)
    assert int(np.argmax(f)) == math.ceil(th / lam) - 1


@pytest.mark.parametrize("lam,B", [(-3, 10), (-1, 4), (-5, 5), (-7, 30)])
def test_negative_branch_linear(oracle_mod, lam, B):
    # G4, LIN: pot_t = -(((t+1)|lam| - 1) mod B + 1) for |lam| <= B, no spikes.
    T = 50
    net = single_neuron(w=0, leak=lam, pos=1000, neg=-B, mode=MODE_LIN)
    f, p, _ = fired_trace(oracle_mod, net, no_input(T=1), T)
    L = -lam
    assert f.sum() == 0
    for t in range(T):
        assert p[t] == -((((t + 1) * L - 1) % B) + 1)


@pytest.mark.parametrize("lam,B", [(-3, 10), (-1, 4), (-5, 5), (-7, 30)])
def test_negative_branch_absolute(oracle_mod, lam, B):
    # G4, ABS with R = 0: reset to 0 when v < -B; period k = floor(B/|lam|)+1.
    T = 50
    net = single_neuron(w=0, leak=lam, pos=1000, neg=-B, reset=0, mode=MODE_ABS)
    _, p, _ = fired_trace(oracle_mod, net, no_input(T=1), T)
    L = -lam
    k = B // L + 1
    for t in range(T):
        m = t % k
        assert p[t] == (0 if m == k - 1 else -(m + 1) * L)


def test_negative_absolute_reset_value(oracle_mod):
    # ABS negative reset goes to -R (G4); R = 7
    net = single_neuron(w=0, leak=-4, pos=1000, neg=-10, reset=7, mode=MODE_ABS)
    _, p, _ = fired_trace(oracle_mod, net, no_input(T=1), 6)
    # -4, -8, -12 < -10 -> -7, -11 -> -7, ...
    assert list(p) == [-4, -8, -7, -7, -7, -7]


def test_saturation(oracle_mod):
    # P3: w = 50 every tick, pb = 8, theta+ = 200: pot = min(50(t+1), 127),
    # never fires (v <= 127 + 50 < 200).
    T = 20
    net = single_neuron(w=50, pos=200, pb=8, mode=MODE_ABS)
    f, p, _ = fired_trace(oracle_mod, net, input_every_tick(T), T)
    assert f.sum() == 0
    assert list(p) == [min(50 * (t + 1), 127) for t in range(T)]


def test_zero_drive_never_fires(oracle_mod):
    # P5: zero input, zero leak, theta+ > initial potential: never fires,
    # potential constant.
    net = single_neuron(w=5, leak=0, pos=10, init=9)
    f, p, _ = fired_trace(oracle_mod, net, no_input(T=1), 40)
    assert f.sum() == 0 and set(p) == {9}


def test_input_arrival_tick(oracle_mod):
    # G8: input at tick t with theta+=1, w=1 fires at t (tick 0 allowed).
    for t0 in (0, 1, 5):
        net = single_neuron(w=1, pos=1)
        f, _, _ = fired_trace(oracle_mod, net, input_at([t0], t0 + 1), t0 + 3)
        assert list(np.nonzero(f)[0]) == [t0]


def test_spec_run_tick_examples(oracle_mod):
    # input visible at tick 1 (SPEC's offset-1 delivery staged on tick 0)
    net = single_neuron(w=1, pos=1)
    _, _, o = fired_trace(oracle_mod, net, input_at([1], 2), 3)
    assert [tuple(e) for e in o.events()] == [(0, 1, 0, 0, 0)]
    # 1x2 relay, core 0 stimulated (arrival tick 1) -> core 1 spikes at tick 2
    net = relay_chain(2, 1)
    o = oracle_mod.Oracle(net, input_at([1], 2)).run(4)
    assert [tuple(e) for e in o.events()] == [(0, 2, 1, 0, 0)]


# --------------------------------------------------------------------------
# delivery at the scheduled tick (P4), scheduler properties
# --------------------------------------------------------------------------

@pytest.mark.parametrize("D", [1, 2, 3, 7, 15])
def test_relay_delivery_every_delay(oracle_mod, D):
    # P4: L-core relay with delay d, input at t0 -> output at t0 + (L-1) d,
    # for every d in 1..D including d = D (catches the SPEC D-row ring, G6).
    L, t0 = 4, 2
    for d in range(1, D + 1):
        net = relay_chain(L, d, D=D)
        T = t0 + (L - 1) * d + 3
        o = oracle_mod.Oracle(net, input_at([t0], t0 + 1)).run(T)
        ev = o.events()
        assert [tuple(e) for e in ev] == [(0, t0 + (L - 1) * d, L - 1, 0, 0)], (d, D)


def test_worked_relay_4_3_2(oracle_mod):
    # P4's worked case: L = 4, d = 3, t0 = 2 -> output at 11.
    o = oracle_mod.Oracle(relay_chain(4, 3), input_at([2], 3)).run(15)
    assert o.events()[:, 1].tolist() == [11]


@pytest.mark.parametrize("D", [1, 4, 15])
def test_offset_k_visibility(oracle_mod, D):
    # a spike sent with offset k is pending exactly k ticks later and
    # never before/after; pending row j holds spikes due at now + j.
    for k in range(1, D + 1):
        net = relay_chain(2, k, D=D)
        o = oracle_mod.Oracle(net, input_at([0], 1))
        o.run(1)                                    # core 0 fires at tick 0
        for elapsed in range(1, k + 1):
            pend = o.pending()[0, 1, :, 0]          # core 1, all rows, axon 0
            row = k - elapsed                       # due at 0 + k = now + row
            want = np.zeros(D, np.uint8)
            want[row] = 1
            assert np.array_equal(pend, want), (k, elapsed)
            o.run(1)
        assert o.pending().sum() == 0               # consumed at tick k
        assert o.fired()[0, 1, 0] == 1


def test_idle_ring_drains(oracle_mod):
    # after D idle ticks with no deliveries the scheduler is empty
    from workloads.gen import config1
    net, inp = config1(T=8)
    o = oracle_mod.Oracle(net, inp).run(8)
    assert o.pending().sum() > 0
    net2 = net.copy()
    net2.pos_threshold[:] = 30000          # nothing fires any more
    o2 = oracle_mod.Oracle(net2, inp).run(net.max_delay + 8)
    assert o2.pending().sum() == 0


def test_determinism(oracle_mod):
    from workloads.gen import corpus_case
    net, inp = corpus_case(3)
    a = oracle_mod.Oracle(net, inp).run(12)
    b = oracle_mod.Oracle(net, inp).run(12)
    assert np.array_equal(a.potentials(), b.potentials())
    assert np.array_equal(a.events(), b.events())
