"""Seeded synthetic workloads shaped like the paper's (Table I).

The paper's trained networks and datasets are not available,
so every workload here is synthetic with the paper's shapes; the recipes are
SURVEY.md 8(d) and DESIGN.md section 5.  Seeds: network = 1000 + config#,
inputs = 2000 + config#, corpus seeds 0..999.

All randomness comes from workloads.rng.SplitMix64 with exact integer draw
semantics.  No arithmetic of the RANC method lives here: these functions only
lay out arrays (and, for VMM, the matrix/vector the closed-form pin needs).
"""
from __future__ import annotations

import numpy as np

from .netdef import (KIND_NONE, KIND_OUTPUT, KIND_ROUTE, MODE_ABS, MODE_LIN,
                     Inputs, Network, words)
from .rng import SplitMix64, substream

# ----------------------------------------------------------------------------
# helpers
# ----------------------------------------------------------------------------


def _blank(grid_w, grid_h, A, N, K, D, C, I, pb=16, wb=9, lb=9, tb=9, rb=9, name="net"):
    G = grid_w * grid_h
    z = lambda dt: np.zeros((G, N), dtype=dt)  # noqa: E731
    return Network(
        grid_w=grid_w, grid_h=grid_h, axons=A, neurons=N, num_types=K, max_delay=D,
        num_classes=C, num_lines=I, potential_bits=pb, weight_bits=wb, leak_bits=lb,
        threshold_bits=tb, reset_bits=rb,
        axon_type=np.zeros((G, A), np.uint8), input_line=np.full((G, A), -1, np.int32),
        crossbar=np.zeros((G, N, words(A)), np.uint32), weight=np.zeros((G, N, K), np.int16),
        leak=z(np.int16), pos_threshold=np.ones((G, N), np.int16), neg_threshold=z(np.int16),
        reset_potential=z(np.int16), initial_potential=z(np.int16), reset_mode=z(np.uint8),
        dest_kind=z(np.uint8), dest_dx=z(np.int16), dest_dy=z(np.int16), dest_axon=z(np.int16),
        dest_delay=np.ones((G, N), np.uint8), out_class=z(np.uint16), name=name)


def perf_params(net: Network, rng: SplitMix64, cores=None, density=0.5):
    """SURVEY 8(d) neuron parameters for perf configs: crossbar density 0.5,
    types uniform, weights U[-8,8] (wb 9), leak U[-2,0], theta+ U[4,32],
    theta- U[-32,-4], R = 0, mode ABS 70% / LIN 30%, pb 16."""
    G, A, N, K = net.G, net.axons, net.neurons, net.num_types
    cores = np.arange(G) if cores is None else np.asarray(cores)
    g = len(cores)
    net.axon_type[cores] = rng.ints(g * A, 0, K - 1).reshape(g, A).astype(np.uint8)
    conn = rng.bernoulli(g * N * A, density).reshape(g, N, A)
    net.crossbar[cores] = Network.pack_conn(conn)
    net.weight[cores] = rng.ints(g * N * K, -8, 8).reshape(g, N, K).astype(np.int16)
    net.leak[cores] = rng.ints(g * N, -2, 0).reshape(g, N)
    net.pos_threshold[cores] = rng.ints(g * N, 4, 32).reshape(g, N)
    net.neg_threshold[cores] = rng.ints(g * N, -32, -4).reshape(g, N)
    net.reset_potential[cores] = 0
    net.initial_potential[cores] = 0
    net.reset_mode[cores] = (rng.ints(g * N, 0, 9) >= 7).reshape(g, N).astype(np.uint8)


def bernoulli_inputs(rng: SplitMix64, S, T_in, I, p) -> Inputs:
    return Inputs.from_dense(rng.bernoulli(S * T_in * I, p).reshape(S, T_in, I))


# ----------------------------------------------------------------------------
# synthetic digits (MNIST-shaped rate-coded input)
# ----------------------------------------------------------------------------


def _stroke(img, rng):
    x0, y0, x1, y1 = (int(v) for v in rng.ints(4, 3, 23))
    L = max(abs(x1 - x0), abs(y1 - y0), 1)
    for k in range(L + 1):
        x = x0 + (x1 - x0) * k // L
        y = y0 + (y1 - y0) * k // L
        img[y:y + 2, x:x + 2] = True


def digit_prototypes(seed=77):
    rng = substream(seed, "digit-prototypes")
    protos = np.zeros((10, 28, 28), bool)
    for c in range(10):
        for _ in range(3):
            _stroke(protos[c], rng)
    return protos


def synthetic_digits(S, T_in, seed, protos=None):
    """S rate-coded 28x28 samples: prototype of class y ~ U{0..9}, shifted by
    U[-2,2] px, 5% pixel flips, 'on' intensity level q ~ U{128..255} giving
    spike probability (q+1)/256 per tick.  Returns (Inputs, labels)."""
    protos = digit_prototypes() if protos is None else protos
    rng = substream(seed, "digits")
    labels = rng.ints(S, 0, 9)
    shifts = rng.ints(2 * S, -2, 2).reshape(S, 2)
    flips = rng.bernoulli(S * 784, 0.05).reshape(S, 28, 28)
    q = rng.ints(S * 784, 128, 255).reshape(S, 784)
    imgs = np.zeros((S, 28, 28), bool)
    for s in range(S):
        imgs[s] = np.roll(protos[labels[s]], (int(shifts[s, 0]), int(shifts[s, 1])), axis=(0, 1))
    imgs ^= flips
    level = np.where(imgs.reshape(S, 784), q, -1)           # -1: never spikes
    spk = np.zeros((S, T_in, 784), bool)
    chunk = 256
    for lo in range(0, S, chunk):
        hi = min(S, lo + chunk)
        n = (hi - lo) * T_in * 784
        u = rng.u64((n + 7) // 8)
        b = u.view(np.uint8)[:n].reshape(hi - lo, T_in, 784).astype(np.int16)
        spk[lo:hi] = b <= level[lo:hi, None, :]
    inp = Inputs.from_dense(spk, labels=labels)
    return inp, labels


def stream_digits(n_images, seed, protos=None):
    """Paper-faithful streaming input (10000 test
    images in 10010 ticks): ONE sample whose input at tick t is image t
    (prototype of class U{0..9}, shifted U[-2,2] px, 5% flips), each 'on'
    pixel spiking once, at that tick.  Returns (Inputs, labels)."""
    protos = digit_prototypes() if protos is None else protos
    rng = substream(seed, "stream-digits")
    labels = rng.ints(n_images, 0, 9)
    shifts = rng.ints(2 * n_images, -2, 2).reshape(n_images, 2)
    flips = rng.bernoulli(n_images * 784, 0.05).reshape(n_images, 28, 28)
    spk = np.zeros((1, n_images, 784), bool)
    for t in range(n_images):
        img = np.roll(protos[labels[t]], (int(shifts[t, 0]), int(shifts[t, 1])), axis=(0, 1)) ^ flips[t]
        spk[0, t] = img.reshape(784)
    return Inputs.from_dense(spk, labels=labels), labels


def config3_stream(n_images=10000, seed=1003, inputs_seed=2013):
    """The config-3 network fed one image per tick (streaming, f2);
    T = n_images + 3 drains the 4-layer pipeline."""
    net, _ = config3(seed=seed, S=0)
    net.name = "config3-stream"
    inp, _ = stream_digits(n_images, inputs_seed)
    net.meta.update(T=n_images + 3)
    return net, inp


def sweep_variants(net, V, seed=3000):
    """V design-space variants of a network:
    variant v scales the positive thresholds by (1 + v/4), shifts the leaks
    by -(v mod 3) and flips the reset mode of a seeded 1/(v+2) fraction of
    neurons; crossbars, weights and routes are shared.  Values stay inside the
    network's bitwidths."""
    import dataclasses
    rng = substream(seed, f"sweep-{net.name}")
    tmax = (1 << (net.threshold_bits - 1)) - 1
    lmin = -(1 << (net.leak_bits - 1))
    out = []
    for v in range(V):
        pt = np.clip(np.asarray(net.pos_threshold, np.int64) * (4 + v) // 4, 1, tmax).astype(np.int16)
        lk = np.clip(np.asarray(net.leak, np.int64) - (v % 3), lmin, None).astype(np.int16)
        flip = rng.bernoulli(net.G * net.neurons, 1.0 / (v + 2)).reshape(net.G, net.neurons)
        rm = np.where(flip, 1 - np.asarray(net.reset_mode), net.reset_mode).astype(np.uint8)
        vn = dataclasses.replace(net, pos_threshold=pt, leak=lk, reset_mode=rm, name=f"{net.name}-v{v}",
                                 meta=dict(net.meta))
        out.append(vn)
    return out


# ----------------------------------------------------------------------------
# config 1: single 256x256 core
# ----------------------------------------------------------------------------


def config1(seed=1001, T=64, S=1):
    rng = substream(seed, "config1")
    A = N = 256
    net = _blank(1, 1, A, N, 4, 15, 10, 256, name="config1-single-core")
    perf_params(net, rng)
    net.input_line[0] = np.arange(A)
    u = rng.ints(N, 0, 9)
    kind = np.where(u < 7, KIND_ROUTE, np.where(u < 9, KIND_OUTPUT, KIND_NONE))
    net.dest_kind[0] = kind
    net.dest_axon[0] = rng.ints(N, 0, A - 1)
    net.dest_delay[0] = rng.ints(N, 1, 15)
    net.out_class[0] = np.arange(N) % 10
    net.meta.update(T=T)
    inp = bernoulli_inputs(substream(seed + 1000, "config1-in"), S, T, 256, 0.1)
    return net, inp


# ----------------------------------------------------------------------------
# config 2: 5-core MNIST-shaped (4 input cores -> 1 output core)
# ----------------------------------------------------------------------------


def config2(seed=1002, S=1000, T_in=16):
    rng = substream(seed, "config2")
    A = N = 256
    net = _blank(5, 1, A, N, 4, 1, 10, 784, name="config2-mnist-5c")
    perf_params(net, rng)
    offs = [(0, 0), (0, 12), (12, 0), (12, 12)]
    for i, (oy, ox) in enumerate(offs):
        yy, xx = np.meshgrid(np.arange(16) + oy, np.arange(16) + ox, indexing="ij")
        net.input_line[i] = (yy * 28 + xx).reshape(-1)
        net.dest_kind[i, :64] = KIND_ROUTE
        net.dest_dx[i, :64] = 4 - i
        net.dest_dy[i, :64] = 0
        net.dest_axon[i, :64] = 64 * i + np.arange(64)
        net.dest_delay[i, :64] = 1
    net.dest_kind[4, :250] = KIND_OUTPUT
    net.out_class[4, :250] = np.arange(250) // 25
    T = T_in + 1
    net.meta.update(T=T)
    inp, _ = synthetic_digits(S, T_in, seed + 1000)
    return net, inp


# ----------------------------------------------------------------------------
# config 3: 512-core MNIST-shaped inference net (the headline)
# ----------------------------------------------------------------------------


def config3_wide(seed=1003, S=10000, scale=16, **kw):
    """The config-3 net with every weight, leak, threshold and reset scaled by
    `scale` (16: weights up to +-128, beyond int8), so integration needs
    13-bit weights while the dynamics stay those of config 3 (a perf workload
    for the tensor-core wide-weight variant)."""
    net, inp = config3(seed=seed, S=S, **kw)
    for f in ("weight", "leak", "pos_threshold", "neg_threshold", "reset_potential", "initial_potential"):
        setattr(net, f, (getattr(net, f).astype(np.int32) * scale).astype(np.int16))
    extra = int(np.ceil(np.log2(scale)))
    net.weight_bits += extra
    net.leak_bits += extra
    net.threshold_bits += extra
    net.reset_bits += extra
    net.name = f"config3-wide-x{scale}"
    return net, inp


def config3_layout():
    """Core coordinates of the 4 layers on the 32x16 grid."""
    W = 32
    L1 = [(y * W + x) for y in range(14) for x in range(W)]                  # 448
    L2 = [(14 * W + x) for x in range(W)] + [(15 * W + x) for x in range(24)]  # 56
    L3 = [(15 * W + x) for x in range(24, 31)]                               # 7
    L4 = [15 * W + 31]                                                        # 1
    return W, 16, [L1, L2, L3, L4]


def config3(seed=1003, S=10000, T_in=16, inputs_seed=2003):
    rng = substream(seed, "config3")
    A = N = 256
    W, H, layers = config3_layout()
    net = _blank(W, H, A, N, 4, 1, 10, 784, name="config3-mnist-512c")
    perf_params(net, rng)
    L1, L2, L3, L4 = layers
    for c1, core in enumerate(L1):
        p = c1 % 16
        oy, ox = 4 * (p // 4), 4 * (p % 4)
        yy, xx = np.meshgrid(np.arange(16) + oy, np.arange(16) + ox, indexing="ij")
        net.input_line[core] = (yy * 28 + xx).reshape(-1)

    def wire(src_layer, dst_layer, stride):
        for c, core in enumerate(src_layer):
            dst = dst_layer[c // stride]
            sx, sy = core % W, core // W
            tx, ty = dst % W, dst // W
            base = 32 * (c % stride)
            net.dest_kind[core, :32] = KIND_ROUTE
            net.dest_dx[core, :32] = tx - sx
            net.dest_dy[core, :32] = ty - sy
            net.dest_axon[core, :32] = base + np.arange(32)
            net.dest_delay[core, :32] = 1

    wire(L1, L2, 8)
    wire(L2, L3, 8)
    wire(L3, L4, 8)      # L3 core c -> L4 axons [32c, +32)
    net.dest_kind[L4[0], :250] = KIND_OUTPUT
    net.out_class[L4[0], :250] = np.arange(250) // 25
    T = T_in + 3
    net.meta.update(T=T, layers=layers)
    inp = None
    if S > 0:
        inp, _ = synthetic_digits(S, T_in, inputs_seed)
    return net, inp


# ----------------------------------------------------------------------------
# config 4: vector-matrix multiply (P6 closed-form mapping)
# ----------------------------------------------------------------------------


def vmm(n, m, Mmax, Xmax, S=1000, seed=1004, A=256, block_in=None, block_out=None):
    """RANC VMM y = M x with 0/1 spike-count coding.

    Input i carries x_i spikes on ticks 0..x_i-1 and feeds 4 axons of types
    0..3 whose per-neuron weights are (1, 2, 4, 8).  Counting neuron j+
    connects the type-k axon of input i iff bit k of max(M_ji, 0) is set
    (j- likewise with max(-M_ji, 0)); theta+ = 1, linear reset, leak 0, so it
    emits exactly (M+ x)_j spikes.  With more inputs than one core's axons,
    partial cores feed adder cores (weight-1 axons, same counting neuron),
    which again emit exactly the sum.  Output class 2j (+) and 2j+1 (-).
    """
    rng = substream(seed, f"vmm-{n}-{m}")
    M = rng.ints(m * n, -Mmax, Mmax).reshape(m, n)
    X = rng.ints(S * n, 0, Xmax).reshape(S, n)
    bin_ = block_in or min(n, A // 4)
    bout = block_out or min(m, 128)
    nb_in = -(-n // bin_)
    nb_out = -(-m // bout)
    two_layer = nb_in > 1
    # adder cores: each handles `per_adder` outputs * 2 signs * nb_in partial axons
    per_adder = max(1, A // (2 * nb_in)) if two_layer else 0
    n_partial = nb_in * nb_out
    n_adder = (-(-m // per_adder)) if two_layer else 0
    G = n_partial + n_adder
    gw = int(np.ceil(np.sqrt(G)))
    gh = -(-G // gw)
    N = 256
    assert 2 * bout <= N and 4 * bin_ <= A
    net = _blank(gw, gh, A, N, 4, 1, 2 * m, n, tb=16, name=f"vmm-{n}x{m}")
    net.neg_threshold[:] = -(1 << 15)
    net.pos_threshold[:] = 1
    net.reset_mode[:] = MODE_LIN
    net.leak[:] = 0
    net.weight[:, :, :] = np.array([1, 2, 4, 8], np.int16)
    Mp, Mn = np.maximum(M, 0), np.maximum(-M, 0)
    conn = np.zeros((net.G, N, A), bool)   # grid may have spare empty cores

    def coord(c):
        return c % gw, c // gw

    for bi in range(nb_in):
        for bo in range(nb_out):
            core = bi * nb_out + bo
            ins = np.arange(bi * bin_, min(n, (bi + 1) * bin_))
            outs = np.arange(bo * bout, min(m, (bo + 1) * bout))
            for li, i in enumerate(ins):
                net.input_line[core, 4 * li:4 * li + 4] = i
                net.axon_type[core, 4 * li:4 * li + 4] = np.arange(4)
            for lj, j in enumerate(outs):
                for sign, Ms in ((0, Mp), (1, Mn)):
                    nrn = 2 * lj + sign
                    for li, i in enumerate(ins):
                        v = Ms[j, i]
                        for k in range(4):
                            if (v >> k) & 1:
                                conn[core, nrn, 4 * li + k] = True
                    if two_layer:
                        ac = n_partial + j // per_adder
                        ax = ((j % per_adder) * 2 + sign) * nb_in + bi
                        sx, sy = coord(core)
                        tx, ty = coord(ac)
                        net.dest_kind[core, nrn] = KIND_ROUTE
                        net.dest_dx[core, nrn] = tx - sx
                        net.dest_dy[core, nrn] = ty - sy
                        net.dest_axon[core, nrn] = ax
                        net.dest_delay[core, nrn] = 1
                    else:
                        net.dest_kind[core, nrn] = KIND_OUTPUT
                        net.out_class[core, nrn] = 2 * j + sign
    for a_i in range(n_adder):
        core = n_partial + a_i
        net.axon_type[core] = 0
        for lj in range(per_adder):
            j = a_i * per_adder + lj
            if j >= m:
                break
            for sign in range(2):
                nrn = 2 * lj + sign
                base = (lj * 2 + sign) * nb_in
                conn[core, nrn, base:base + nb_in] = True
                net.dest_kind[core, nrn] = KIND_OUTPUT
                net.out_class[core, nrn] = 2 * j + sign
    net.crossbar[:] = Network.pack_conn(conn)
    spk = np.zeros((S, Xmax, n), bool)
    for t in range(Xmax):
        spk[:, t, :] = X > t
    inp = Inputs.from_dense(spk)
    y_max = int(max((Mp @ X.T).max(initial=0), (Mn @ X.T).max(initial=0)))
    # drain bound: a counting neuron is a unit-rate queue, so its last spike is
    # at most (last arrival) + (its total count).  Single layer: Xmax-1+y_max;
    # adder layer: (Xmax-1+y_max) + 1 + y_max.
    T = (Xmax + 2 * y_max + 2) if two_layer else (Xmax + y_max + 1)
    net.meta.update(M=M, X=X, T=T, two_layer=two_layer)
    return net, inp


VMM_VARIANTS = {
    "vmm32": dict(n=32, m=32, Mmax=15, Xmax=15, A=256),
    "vmm60": dict(n=60, m=60, Mmax=15, Xmax=15, A=512),
    "vmm256": dict(n=256, m=256, Mmax=15, Xmax=7, A=256),
    "vmm1024": dict(n=1024, m=1024, Mmax=3, Xmax=7, A=256),
}


def config4(variant="vmm32", S=1000, seed=1004):
    return vmm(S=S, seed=seed, **VMM_VARIANTS[variant])


# ----------------------------------------------------------------------------
# config 5: 4096-core random 2-D mesh (TrueNorth-Ref-shaped)
# ----------------------------------------------------------------------------


def config5(seed=1005, S=64, T=500, grid=64, variant="local", drive=True):
    rng = substream(seed, f"config5-{variant}")
    A = N = 256
    net = _blank(grid, grid, A, N, 4, 15, 10, 0, name=f"config5-mesh-{grid}x{grid}-{variant}")
    perf_params(net, rng, density=0.25)
    G = net.G
    u = rng.ints(G * N, 0, 99).reshape(G, N)
    kind = np.where(u < 94, KIND_ROUTE, np.where(u < 95, KIND_OUTPUT, KIND_NONE))
    net.dest_kind[:] = kind
    x = (np.arange(G) % grid)[:, None]
    y = (np.arange(G) // grid)[:, None]
    if variant == "local":
        dx = rng.ints(G * N, -4, 4).reshape(G, N)
        dy = rng.ints(G * N, -4, 4).reshape(G, N)
        tx, ty = x + dx, y + dy
        tx = np.where(tx < 0, -tx, np.where(tx >= grid, 2 * (grid - 1) - tx, tx))
        ty = np.where(ty < 0, -ty, np.where(ty >= grid, 2 * (grid - 1) - ty, ty))
    else:
        tx = rng.ints(G * N, 0, grid - 1).reshape(G, N)
        ty = rng.ints(G * N, 0, grid - 1).reshape(G, N)
    route = kind == KIND_ROUTE
    net.dest_dx[:] = np.where(route, tx - x, 0)
    net.dest_dy[:] = np.where(route, ty - y, 0)
    net.dest_axon[:] = rng.ints(G * N, 0, A - 1).reshape(G, N)
    net.dest_delay[:] = rng.ints(G * N, 1, 15).reshape(G, N)
    net.out_class[:] = (np.arange(N) % 10)[None, :]
    if drive:
        on = rng.bernoulli(G * N, 0.10).reshape(G, N)
        net.leak[:] = np.where(on, rng.ints(G * N, 1, 4).reshape(G, N), net.leak)
    else:
        net.leak[:] = 0
    net.meta.update(T=T)
    inp = Inputs(S, 0, np.zeros((S, 0, 0), np.uint32))
    return net, inp


# ----------------------------------------------------------------------------
# random tiny / corpus networks (parity corpus, brute force)
# ----------------------------------------------------------------------------


def random_network(seed, grid_w, grid_h, A, N, K, D, C=None, I=None, density=0.5,
                   pb=16, wb=9, lb=9, tb=9, rb=9, full_range=True, route_frac=0.6,
                   out_frac=0.25, input_frac=0.5):
    """Random network with full-range parameters (stress corpus)."""
    rng = substream(seed, "random-network")
    C = C if C is not None else 3
    I = I if I is not None else max(1, A // 2)
    net = _blank(grid_w, grid_h, A, N, K, D, C, I, pb, wb, lb, tb, rb, name=f"rand-{seed}")
    G = net.G

    def srange(bits, n, frac=1.0):
        hi = (1 << (bits - 1)) - 1
        lo = -(1 << (bits - 1))
        if not full_range:
            hi, lo = max(1, int(hi * frac)), min(-1, int(lo * frac))
        return rng.ints(n, lo, hi)

    net.axon_type[:] = rng.ints(G * A, 0, K - 1).reshape(G, A)
    il = rng.ints(G * A, 0, I - 1).reshape(G, A)
    use = rng.bernoulli(G * A, input_frac).reshape(G, A)
    net.input_line[:] = np.where(use, il, -1)
    conn = rng.bernoulli(G * N * A, density).reshape(G, N, A)
    net.crossbar[:] = Network.pack_conn(conn)
    net.weight[:] = srange(wb, G * N * K).reshape(G, N, K)
    net.leak[:] = srange(lb, G * N, 0.1).reshape(G, N)
    th_hi = (1 << (tb - 1)) - 1
    th_lo = -(1 << (tb - 1))
    pos = rng.ints(G * N, 0, th_hi).reshape(G, N)
    neg = rng.ints(G * N, th_lo, 0).reshape(G, N)
    # a fraction of neurons gets small thresholds so that they fire often
    small = rng.bernoulli(G * N, 0.5).reshape(G, N)
    pos = np.where(small, rng.ints(G * N, 1, 8).reshape(G, N), pos)
    neg = np.where(small, rng.ints(G * N, -8, -1).reshape(G, N), neg)
    net.pos_threshold[:] = pos
    net.neg_threshold[:] = neg
    net.reset_potential[:] = rng.ints(G * N, 0, (1 << (rb - 1)) - 1).reshape(G, N)
    net.initial_potential[:] = srange(pb, G * N).reshape(G, N)
    net.reset_mode[:] = rng.ints(G * N, 0, 1).reshape(G, N)
    u = rng.ints(G * N, 0, 999).reshape(G, N)
    kind = np.where(u < route_frac * 1000, KIND_ROUTE,
                    np.where(u < (route_frac + out_frac) * 1000, KIND_OUTPUT, KIND_NONE))
    net.dest_kind[:] = kind
    x = (np.arange(G) % grid_w)[:, None]
    y = (np.arange(G) // grid_w)[:, None]
    tx = rng.ints(G * N, 0, grid_w - 1).reshape(G, N)
    ty = rng.ints(G * N, 0, grid_h - 1).reshape(G, N)
    route = kind == KIND_ROUTE
    net.dest_dx[:] = np.where(route, tx - x, 0)
    net.dest_dy[:] = np.where(route, ty - y, 0)
    net.dest_axon[:] = rng.ints(G * N, 0, A - 1).reshape(G, N)
    # delays: uniform, with extra mass on delay == D (G6 corner)
    dl = rng.ints(G * N, 1, D).reshape(G, N)
    atD = rng.bernoulli(G * N, 0.25).reshape(G, N)
    net.dest_delay[:] = np.where(atD, D, dl)
    net.out_class[:] = rng.ints(G * N, 0, max(C, 1) - 1).reshape(G, N)
    if C == 0:
        net.dest_kind[:] = np.where(kind == KIND_OUTPUT, KIND_NONE, kind)
    return net


def random_inputs(seed, net: Network, S, T_in, p=0.3) -> Inputs:
    rng = substream(seed, "random-inputs")
    return bernoulli_inputs(rng, S, T_in, net.num_lines, p)


def tiny_case(seed):
    """Random tiny mesh for brute force (<= 2x2 cores, <= 8 axons/neurons,
    K <= 4, D <= 4, 1-4 samples)."""
    r = substream(seed, "tiny-shape")
    gw, gh = (int(v) for v in r.ints(2, 1, 2))
    A, N = (int(v) for v in r.ints(2, 1, 8))
    K = int(r.ints(1, 1, 4)[0])
    D = int(r.ints(1, 1, 4)[0])
    S = int(r.ints(1, 1, 4)[0])
    pb = int([4, 8, 12, 16][int(r.ints(1, 0, 3)[0])])
    wb = int(r.ints(1, 2, 9)[0])
    I = int(r.ints(1, 1, 6)[0])
    net = random_network(seed, gw, gh, A, N, K, D, C=3, I=I, pb=pb, wb=wb,
                         lb=min(wb, 6), tb=9, rb=min(pb, 9))
    inp = random_inputs(seed, net, S, 20, p=0.4)
    return net, inp


def corpus_case(seed):
    """Parity corpus case: mid-size meshes, A/N not multiples of 32, K < 4,
    delay == D, fan-in collisions, saturation, both reset modes."""
    r = substream(seed, "corpus-shape")
    gw = int(r.ints(1, 1, 4)[0])
    gh = int(r.ints(1, 1, 3)[0])
    A = int([1, 7, 31, 32, 33, 64, 100, 256, 300][int(r.ints(1, 0, 8)[0])])
    N = int([1, 5, 31, 32, 33, 64, 129, 256][int(r.ints(1, 0, 7)[0])])
    K = int(r.ints(1, 1, 4)[0])
    D = int(r.ints(1, 1, 15)[0])
    pb = int([4, 8, 12, 16][int(r.ints(1, 0, 3)[0])])
    wb = int(r.ints(1, 2, 12)[0])
    dens = [0.0, 0.1, 0.5, 1.0][int(r.ints(1, 0, 3)[0])]
    S = int(r.ints(1, 1, 70)[0])
    net = random_network(seed, gw, gh, A, N, K, D, C=4, I=max(1, A), density=dens,
                         pb=pb, wb=wb, lb=min(wb, 8), tb=min(16, max(wb, 9)), rb=min(pb, 12))
    inp = random_inputs(seed, net, S, 12, p=[0.0, 0.01, 0.1, 0.4][int(r.ints(1, 0, 3)[0])])
    return net, inp


CONFIGS = {
    1: config1,
    2: config2,
    3: config3,
    4: config4,
    5: config5,
}


def envelope_case(seed):
    """Configurable-envelope corpus (configurable axons and
    neurons per core and bitwidths): A and N beyond 256 up to the ABI's 1024,
    weights over the FULL range of 13..16 bits, potential widths down to 2
    and 3 bits (saturating almost every tick), K 1..4, D up to 15.  Sizes are
    bounded so the serial oracle finishes in seconds."""
    r = substream(seed, "envelope-shape")
    A = int([513, 1000, 1024, 256, 700, 33][int(r.ints(1, 0, 5)[0])])
    N = int([257, 1000, 1024, 256, 300, 64][int(r.ints(1, 0, 5)[0])])
    wb = int(r.ints(1, 13, 16)[0])
    pb = int([2, 3, 5, 16][int(r.ints(1, 0, 3)[0])])
    K = int(r.ints(1, 1, 4)[0])
    D = int(r.ints(1, 1, 15)[0])
    big = A * N > 300000
    gw = 1 if big else int(r.ints(1, 1, 2)[0])
    gh = int(r.ints(1, 1, 2)[0])
    S = int(r.ints(1, 1, 12 if big else 40)[0])
    dens = [0.1, 0.5, 1.0][int(r.ints(1, 0, 2)[0])]
    net = random_network(7000 + seed, gw, gh, A, N, K, D, C=5, I=max(1, A // 2), density=dens,
                         pb=pb, wb=wb, lb=min(wb, 10), tb=16, rb=min(pb, 12))
    net.name = f"envelope-{seed}-A{A}-N{N}-wb{wb}-pb{pb}"
    # the extremes of the weight range on some synapses of every core
    lo, hi = -(1 << (wb - 1)), (1 << (wb - 1)) - 1
    net.weight[:, 0, :] = lo
    net.weight[:, min(1, N - 1), :] = hi
    inp = random_inputs(7000 + seed, net, S, 8, p=[0.05, 0.2, 0.5][int(r.ints(1, 0, 2)[0])])
    return net, inp


def bigcore(seed=1006, S=4096, T=20, A=512, N=1024, grid=4):
    """Cores beyond the paper's 256x256 (configurable axons / neurons, P:42,
    P:362): a grid x grid mesh of A-axon, N-neuron cores with the perf
    parameter recipe, random routes inside the mesh (D = 15), Bernoulli(0.1)
    inputs on A/2 lines for T_in = T ticks."""
    rng = substream(seed, "bigcore")
    net = _blank(grid, grid, A, N, 4, 15, 10, A // 2, name=f"bigcore-{grid}x{grid}-A{A}-N{N}")
    perf_params(net, rng, density=0.5)
    G = net.G
    il = rng.ints(G * A, 0, A // 2 - 1).reshape(G, A)
    net.input_line[:] = np.where(rng.bernoulli(G * A, 0.5).reshape(G, A), il, -1)
    u = rng.ints(G * N, 0, 99).reshape(G, N)
    kind = np.where(u < 60, KIND_ROUTE, np.where(u < 70, KIND_OUTPUT, KIND_NONE))
    net.dest_kind[:] = kind
    x = (np.arange(G) % grid)[:, None]
    y = (np.arange(G) // grid)[:, None]
    route = kind == KIND_ROUTE
    net.dest_dx[:] = np.where(route, rng.ints(G * N, 0, grid - 1).reshape(G, N) - x, 0)
    net.dest_dy[:] = np.where(route, rng.ints(G * N, 0, grid - 1).reshape(G, N) - y, 0)
    net.dest_axon[:] = rng.ints(G * N, 0, A - 1).reshape(G, N)
    net.dest_delay[:] = rng.ints(G * N, 1, 15).reshape(G, N)
    net.out_class[:] = (np.arange(N) % 10)[None, :]
    net.meta.update(T=T)
    return net, bernoulli_inputs(substream(seed + 1000, "bigcore-inputs"), S, T, A // 2, 0.1)
