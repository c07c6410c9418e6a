"""The G21 state digest of the oracle: an instrument for
per-tick parity at sizes where full state dumps are too large.  Pinned
against a NumPy re-evaluation from the oracle's own state readers (which are
themselves pinned elsewhere) and by its invariances: order-free sums, every
component contributes, and equal states give equal digests."""
import numpy as np

from workloads.gen import config2, tiny_case

M64 = (1 << 64) - 1
K1, K2 = 0x243F6A8885A308D3, 0x13198A2E03707344


def mix(x):
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def numpy_digest(net, pot, fired, spk_in):
    out = []
    G, N, A = net.G, net.neurons, net.axons
    for s in range(pot.shape[0]):
        d = 0
        for c in range(G):
            for n in range(N):
                cn = c * N + n
                d += mix((cn << 32) | (int(pot[s, c, n]) & 0xFFFFFFFF))
                if fired[s, c, n]:
                    d += mix(K1 ^ cn)
            for a in range(A):
                if spk_in[s, c, a]:
                    d += mix(K2 ^ (c * A + a))
        out.append(d & M64)
    return np.array(out, np.uint64)


def test_digest_matches_numpy_each_tick(oracle_mod):
    net, inp = tiny_case(3)
    o = oracle_mod.Oracle(net, inp)
    # spk_in of tick t = the pending row due at t just before the tick, plus inputs;
    # reconstructed independently: rows due now before the tick OR input lines
    for t in range(8):
        before = o.pending()[:, :, 0, :].astype(bool)   # row due at tick t (routes only)
        o.run(1)
        lines = np.zeros_like(before)
        if t < inp.num_input_ticks and net.num_lines:
            bits = inp.line_bits[:, t, :]
            for c in range(net.G):
                for a in range(net.axons):
                    ln = int(net.input_line[c, a])
                    if ln >= 0:
                        lines[:, c, a] = (bits[:, ln >> 5] >> (ln & 31)) & 1
        spk_in = before | lines
        want = numpy_digest(net, o.potentials(), o.fired(), spk_in)
        assert np.array_equal(o.digest(), want), f"tick {t}"


def test_digest_sensitivity_and_sample_independence(oracle_mod):
    net, inp = config2(S=4)
    a = oracle_mod.Oracle(net, inp).run(5).digest()
    b = oracle_mod.Oracle(net, inp.slice(2, 4)).run(5).digest()
    assert np.array_equal(a[2:], b)                      # per-sample, batch-independent
    c = oracle_mod.Oracle(net, inp).run(6).digest()
    assert not np.array_equal(a, c)                      # moves with the state
