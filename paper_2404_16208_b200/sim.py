"""Thin Python binding over the C ABI (include/ranc.h).

Argument marshalling only: every step of the simulation runs in libranc.so's
CUDA kernels.  PyTorch is used for what it is good at here -- the device
caching allocator (optional, via ranc_set_allocator), CUDA streams
(ranc_set_stream) and process groups (NCCL unique-id exchange).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

_NET_ARRAYS = [
    ("axon_type", np.uint8), ("input_line", np.int32), ("crossbar", np.uint32), ("weight", np.int16),
    ("leak", np.int16), ("pos_threshold", np.int16), ("neg_threshold", np.int16),
    ("reset_potential", np.int16), ("initial_potential", np.int16), ("reset_mode", np.uint8),
    ("dest_kind", np.uint8), ("dest_dx", np.int16), ("dest_dy", np.int16), ("dest_axon", np.int16),
    ("dest_delay", np.uint8), ("out_class", np.uint16)]
_NET_INTS = ["grid_w", "grid_h", "axons", "neurons", "num_types", "max_delay", "num_classes", "num_lines",
             "potential_bits", "weight_bits", "leak_bits", "threshold_bits", "reset_bits"]


def _check(lib, status, ctx=None):
    if status != 0:
        msg = lib.ranc_last_error(ctx)
        raise L.RancError(status, msg.decode() if msg else "")


def make_network_desc(net):
    """Build a ranc_network_desc from any object with the named fields.
    Returns (desc, keepalive)."""
    d = L.NetworkDesc()
    d.abi_version = L.RANC_ABI_VERSION
    for n in _NET_INTS:
        setattr(d, n, int(getattr(net, n)))
    keep = []
    for n, dt in _NET_ARRAYS:
        a = np.ascontiguousarray(getattr(net, n), dtype=dt)
        keep.append(a)
        setattr(d, n, a.ctypes.data)
    return d, keep


class Simulator:
    """One libranc context: a network compiled onto one GPU."""

    def __init__(self, net, device: int = 0, stream=None, torch_allocator: bool = False):
        self.lib = L.load()
        self.net = net
        self.device = device
        desc, keep = make_network_desc(net)
        h = C.c_void_p()
        _check(self.lib, self.lib.ranc_load_network(C.byref(desc), device, C.byref(h)))
        self.h = h
        self.S = 0
        self._cb = None
        if stream is not None:
            self.set_stream(stream)
        if torch_allocator:
            self.use_torch_allocator()

    # -- plumbing -----------------------------------------------------------
    def _ck(self, status):
        _check(self.lib, status, self.h)

    def set_stream(self, stream):
        """stream: a torch.cuda.Stream, an int cudaStream_t, or None."""
        ptr = getattr(stream, "cuda_stream", stream)
        self._ck(self.lib.ranc_set_stream(self.h, C.c_void_p(ptr) if ptr else None))
        self._stream = stream if hasattr(stream, "cuda_stream") else None

    def use_torch_allocator(self):
        import torch

        dev = self.device
        stream = getattr(self, "_stream", None)   # blocks belong to the context's stream

        def _alloc(nbytes, _user):
            if stream is not None:
                return torch.cuda.caching_allocator_alloc(int(nbytes), device=dev, stream=stream)
            return torch.cuda.caching_allocator_alloc(int(nbytes), device=dev)

        def _free(ptr, _user):
            torch.cuda.caching_allocator_delete(int(ptr))

        self._cb = (L.ALLOC_FN(_alloc), L.FREE_FN(_free))
        self._ck(self.lib.ranc_set_allocator(self.h, self._cb[0], self._cb[1], None))

    def set_option(self, option: int, value: int):
        self._ck(self.lib.ranc_set_option(self.h, int(option), int(value)))

    def info(self) -> dict:
        i = L.Info()
        self._ck(self.lib.ranc_get_info(self.h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in L.Info._fields_}

    # -- the four calls of the north star -------------------------------------
    def load_inputs(self, inputs):
        lb = np.ascontiguousarray(inputs.line_bits, dtype=np.uint32)
        self._lb = lb
        d = L.InputsDesc()
        d.num_samples = int(inputs.num_samples)
        d.first_sample = int(getattr(inputs, "first_sample", 0))
        d.num_input_ticks = int(inputs.num_input_ticks)
        d.line_bits = lb.ctypes.data if lb.size else None
        self._ck(self.lib.ranc_load_inputs(self.h, C.byref(d)))
        self.S = d.num_samples
        return self

    def reset(self):
        self._ck(self.lib.ranc_reset_state(self.h))
        return self

    def run(self, ticks: int):
        self._ck(self.lib.ranc_run_ticks(self.h, int(ticks)))
        return self

    def outputs(self, out=None) -> np.ndarray:
        C_ = int(self.net.num_classes)
        if out is None:
            out = np.zeros((self.S, C_), np.int32)
        self._ck(self.lib.ranc_read_outputs(self.h, out.ctypes.data if out.size else None, out.size))
        return out

    # -- parity / debug readers ---------------------------------------------
    @property
    def now(self) -> int:
        t = C.c_int64()
        self._ck(self.lib.ranc_now(self.h, C.byref(t)))
        return t.value

    @property
    def cores_local(self) -> int:
        return self.info()["cores_local"]

    def potentials(self) -> np.ndarray:
        """int32 [S][G_local][N] (G_local = G unless core-sharded)."""
        n = self.net
        out = np.zeros((self.S, self.cores_local, n.neurons), np.int32)
        self._ck(self.lib.ranc_read_potentials(self.h, out.ctypes.data, out.size))
        return out

    def pending_words(self) -> np.ndarray:
        n = self.net
        W = (n.axons + 31) // 32
        out = np.zeros((self.S, self.cores_local, n.max_delay, W), np.uint32)
        self._ck(self.lib.ranc_read_pending(self.h, out.ctypes.data, out.size))
        return out

    def pending(self) -> np.ndarray:
        """uint8 [S][G][D][A]: row j = spikes due at tick now + j."""
        w = self.pending_words()
        bits = np.unpackbits(w.view(np.uint8), axis=-1, bitorder="little")
        return bits[..., :self.net.axons]

    def set_trace(self, flags: int):
        self._ck(self.lib.ranc_set_trace(self.h, int(flags)))

    def _trace_bytes(self, kind):
        need = C.c_size_t(0)
        st = self.lib.ranc_read_trace(self.h, kind, None, 0, C.byref(need))
        if st not in (0, 8):
            self._ck(st)
        return need.value

    def raster(self) -> np.ndarray:
        """uint8 [ticks][S][G][N] fired bits of the last run() call."""
        n = self.net
        nb = self._trace_bytes(L.TRACE_SPIKE_RASTER)
        buf = np.zeros(max(nb // 4, 1), np.uint32)
        got = C.c_size_t(0)
        self._ck(self.lib.ranc_read_trace(self.h, L.TRACE_SPIKE_RASTER, buf.ctypes.data, buf.nbytes,
                                          C.byref(got)))
        Wn = (n.neurons + 31) // 32
        w = buf[:nb // 4].reshape(-1, self.S, self.cores_local, Wn)
        bits = np.unpackbits(w.view(np.uint8), axis=-1, bitorder="little")
        return bits[..., :n.neurons]

    def events(self) -> np.ndarray:
        nb = self._trace_bytes(L.TRACE_OUTPUT_EVENTS)
        buf = np.zeros(max(nb // 8, 1), np.int64)
        got = C.c_size_t(0)
        self._ck(self.lib.ranc_read_trace(self.h, L.TRACE_OUTPUT_EVENTS, buf.ctypes.data, buf.nbytes,
                                          C.byref(got)))
        return buf[:nb // 8].reshape(-1, 5)

    def digests(self) -> np.ndarray:
        """uint64 [ticks][S] state digests (RANC_TRACE_STATE_DIGEST)
        of the last run() call."""
        nb = self._trace_bytes(L.TRACE_STATE_DIGEST)
        buf = np.zeros(max(nb // 8, 1), np.uint64)
        got = C.c_size_t(0)
        self._ck(self.lib.ranc_read_trace(self.h, L.TRACE_STATE_DIGEST, buf.ctypes.data, buf.nbytes,
                                          C.byref(got)))
        return buf[:nb // 8].reshape(-1, self.S)

    # -- multi-GPU ----------------------------------------------------------
    @staticmethod
    def unique_id() -> bytes:
        lib = L.load()
        b = (C.c_char * 128)()
        _check(lib, lib.ranc_comm_unique_id(b))
        return bytes(b)

    def comm_init(self, uid: bytes, world: int, rank: int, mode: int = L.SHARD_SAMPLES):
        b = (C.c_char * 128).from_buffer_copy(uid)
        self._ck(self.lib.ranc_comm_init(self.h, b, int(world), int(rank), int(mode)))

    @staticmethod
    def init_loopback(sims, mode: int = L.SHARD_CORES):
        """Make `sims` (one process, one GPU) the ranks of a core-sharded run."""
        arr = (C.c_void_p * len(sims))(*[s.h.value for s in sims])
        _check(sims[0].lib, sims[0].lib.ranc_comm_init_loopback(arr, len(sims), int(mode)), sims[0].h)

    @staticmethod
    def run_loopback(sims, ticks: int):
        arr = (C.c_void_p * len(sims))(*[s.h.value for s in sims])
        _check(sims[0].lib, sims[0].lib.ranc_run_ticks_loopback(arr, len(sims), int(ticks)), sims[0].h)

    def gather_outputs(self, total_samples: int, root: int = 0, rank: int = 0):
        """Sample mode: the [total_samples][C] counts of all ranks' contiguous
        shards (one ncclGather); core mode: pass total_samples = S, returns the
        [S][C] sum.  None off-root.  Every rank passes the same total."""
        C_ = int(self.net.num_classes)
        out = np.zeros((total_samples, C_), np.int32) if rank == root else None
        self._ck(self.lib.ranc_gather_outputs(self.h, out.ctypes.data if out is not None else None,
                                              total_samples * C_, int(root)))
        return out

    @staticmethod
    def plan_core_shards(net, world: int, rank: int) -> dict:
        """Host-only core-sharded plan (ranc_plan_core_shards; no GPU needed):
        this rank's core band and, per peer, the local ids of the cores it
        sends fired bits of and the global ids of the peer cores it receives."""
        lib = L.load()
        desc, keep = make_network_desc(net)
        i32 = C.c_int32
        lo, gl = i32(), i32()
        sc, rc = (i32 * world)(), (i32 * world)()
        cap = int(net.G) * world
        sl, rl = (i32 * max(cap, 1))(), (i32 * max(cap, 1))()
        _check(lib, lib.ranc_plan_core_shards(C.byref(desc), int(world), int(rank), C.byref(lo), C.byref(gl), sc, rc,
                                              sl, cap, rl, cap))
        send, recv, a, b = [], [], 0, 0
        for p in range(world):
            send.append(list(sl[a:a + sc[p]]))
            recv.append(list(rl[b:b + rc[p]]))
            a += sc[p]
            b += rc[p]
        return {"core_lo": lo.value, "cores_local": gl.value, "send": send, "recv": recv}

    # -- lifetime -----------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            self.lib.ranc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
