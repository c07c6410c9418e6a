"""ctypes wrapper of the C oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product
package.  It imports nothing from paper_2404_16208_b200.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")


def build(force=False) -> str:
    """Compile the oracle with plain gcc -O2 (no vectorisation flags)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", LIB, SRC])
    return LIB


class _Net(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "grid_w", "grid_h", "axons", "neurons", "num_types", "max_delay",
        "num_classes", "num_lines", "potential_bits")] + [
        ("axon_type", C.c_void_p), ("input_line", C.c_void_p), ("crossbar", C.c_void_p),
        ("weight", C.c_void_p), ("leak", C.c_void_p), ("pos_threshold", C.c_void_p),
        ("neg_threshold", C.c_void_p), ("reset_potential", C.c_void_p),
        ("initial_potential", C.c_void_p), ("reset_mode", C.c_void_p),
        ("dest_kind", C.c_void_p), ("dest_dx", C.c_void_p), ("dest_dy", C.c_void_p),
        ("dest_axon", C.c_void_p), ("dest_delay", C.c_void_p), ("out_class", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_saturate.restype = C.c_int64
        _lib.oracle_saturate.argtypes = [C.c_int64, C.c_int]
        _lib.oracle_integrate.restype = C.c_int64
        _lib.oracle_integrate.argtypes = [C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        _lib.oracle_lif.restype = C.c_int64
        _lib.oracle_lif.argtypes = [C.c_int64] * 5 + [C.c_int, C.c_int, C.POINTER(C.c_int)]
        _lib.oracle_create.restype = C.c_void_p
        _lib.oracle_create.argtypes = [C.POINTER(_Net), C.c_int32, C.c_int32, C.c_void_p]
        _lib.oracle_destroy.argtypes = [C.c_void_p]
        _lib.oracle_run.argtypes = [C.c_void_p, C.c_int64]
        _lib.oracle_now.restype = C.c_int64
        _lib.oracle_now.argtypes = [C.c_void_p]
        for f in ("oracle_get_potentials", "oracle_get_pending", "oracle_get_fired",
                  "oracle_get_counts", "oracle_digest"):
            getattr(_lib, f).argtypes = [C.c_void_p, C.c_void_p]
        _lib.oracle_get_events.restype = C.c_int64
        _lib.oracle_get_events.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    return _lib


def saturate(v, bits):
    return lib().oracle_saturate(int(v), int(bits))


def integrate(pot, spikes, conn, types, w):
    A = len(spikes)
    sp = np.ascontiguousarray(spikes, np.uint8)
    cn = np.ascontiguousarray(conn, np.uint8)
    ty = np.ascontiguousarray(types, np.uint8)
    ww = np.ascontiguousarray(w, np.int64)
    return lib().oracle_integrate(int(pot), A, sp.ctypes.data, cn.ctypes.data,
                                  ty.ctypes.data, ww.ctypes.data)


def lif(integrated, leak, pos_th, neg_th, reset, mode, pb):
    f = C.c_int(0)
    v = lib().oracle_lif(int(integrated), int(leak), int(pos_th), int(neg_th), int(reset),
                         int(mode), int(pb), C.byref(f))
    return v, bool(f.value)


class Oracle:
    """Serial oracle over S independent samples; step with run(k)."""

    def __init__(self, net, inputs):
        self.net, self.inputs = net, inputs
        L = lib()
        self._keep = [net, inputs]
        s = _Net()
        for n in ("grid_w", "grid_h", "axons", "neurons", "num_types", "max_delay",
                  "num_classes", "num_lines", "potential_bits"):
            setattr(s, n, int(getattr(net, n)))
        for n, _ in _Net._fields_[9:]:
            setattr(s, n, getattr(net, n).ctypes.data)
        self._s = s
        lb = inputs.line_bits
        if lb.size == 0:
            lb = np.zeros(1, np.uint32)
        self._lb = np.ascontiguousarray(lb, np.uint32)
        self.S = inputs.num_samples
        self.h = L.oracle_create(C.byref(s), self.S, inputs.num_input_ticks, self._lb.ctypes.data)
        if not self.h:
            raise ValueError("oracle_create failed")

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_destroy(self.h)
            self.h = None

    def run(self, ticks: int):
        lib().oracle_run(self.h, int(ticks))
        return self

    @property
    def now(self):
        return lib().oracle_now(self.h)

    def potentials(self):
        n = self.net
        out = np.zeros((self.S, n.G, n.neurons), np.int64)
        lib().oracle_get_potentials(self.h, out.ctypes.data)
        return out

    def pending(self):
        """uint8 [S][G][D][A]; row j = spikes due at tick now+j."""
        n = self.net
        out = np.zeros((self.S, n.G, n.max_delay, n.axons), np.uint8)
        lib().oracle_get_pending(self.h, out.ctypes.data)
        return out

    def fired(self):
        n = self.net
        out = np.zeros((self.S, n.G, n.neurons), np.uint8)
        lib().oracle_get_fired(self.h, out.ctypes.data)
        return out

    def counts(self):
        out = np.zeros((self.S, max(self.net.num_classes, 0)), np.int64)
        if out.size:
            lib().oracle_get_counts(self.h, out.ctypes.data)
        return out

    def digest(self):
        """SURVEY G21 state digest of the last executed tick, uint64 [S]."""
        out = np.zeros(self.S, np.uint64)
        lib().oracle_digest(self.h, out.ctypes.data)
        return out

    def events(self):
        total = lib().oracle_get_events(self.h, None, 0)
        out = np.zeros((max(total, 1), 5), np.int64)
        lib().oracle_get_events(self.h, out.ctypes.data, total)
        return out[:total]
