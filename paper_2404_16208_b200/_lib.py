"""ctypes declarations of include/ranc.h (argument marshalling only).

Loading fails loudly if libranc.so is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RANC_LIB") or os.path.join(PKG, "libranc.so")   # RANC_LIB: A/B builds

RANC_ABI_VERSION = 1
STATUS = {0: "RANC_OK", 1: "RANC_E_ARG", 2: "RANC_E_CONFIG", 3: "RANC_E_BITWIDTH", 4: "RANC_E_RANGE",
          5: "RANC_E_OFFGRID", 6: "RANC_E_BOUND", 7: "RANC_E_STATE", 8: "RANC_E_SIZE", 9: "RANC_E_CUDA",
          10: "RANC_E_OOM", 11: "RANC_E_NCCL"}
TRACE_SPIKE_RASTER = 1
TRACE_OUTPUT_EVENTS = 2
TRACE_STATE_DIGEST = 4
OPT_SAMPLE_TILE = 1
OPT_INPUT_DECODE = 2
OPT_KERNEL = 3
OPT_STREAM = 4
OPT_RING_LAYOUT = 5
OPT_DEBUG_FAULT = 6   # mutation tests only (changes results)
OPT_OPERAND = 7
SHARD_SAMPLES = 0
SHARD_CORES = 1


class RancError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        self.code = STATUS.get(status, str(status))
        super().__init__(f"{self.code}: {msg}")


class NetworkDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "abi_version", "grid_w", "grid_h", "axons", "neurons", "num_types", "max_delay", "num_classes",
        "num_lines", "potential_bits", "weight_bits", "leak_bits", "threshold_bits", "reset_bits")] + [
        (n, C.c_void_p) for n in (
            "axon_type", "input_line", "crossbar", "weight", "leak", "pos_threshold", "neg_threshold",
            "reset_potential", "initial_potential", "reset_mode", "dest_kind", "dest_dx", "dest_dy",
            "dest_axon", "dest_delay", "out_class")]


class InputsDesc(C.Structure):
    _fields_ = [("num_samples", C.c_int32), ("first_sample", C.c_int64), ("num_input_ticks", C.c_int32),
                ("line_bits", C.c_void_p)]


class Info(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "grid_w", "grid_h", "axons", "neurons", "num_types", "max_delay", "num_classes", "num_lines",
        "ring_rows", "ring_words", "pieces", "sample_tile")] + [
        ("num_samples", C.c_int64), ("device_bytes", C.c_int64), ("kernel_launches", C.c_int64),
        ("kernel", C.c_int32), ("core_lo", C.c_int32), ("cores_local", C.c_int32), ("shard_mode", C.c_int32),
        ("exchange_bytes", C.c_int64), ("ring_layout", C.c_int32), ("operand", C.c_int32)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)

EXPORTS = [
    "ranc_load_network", "ranc_load_inputs", "ranc_reset_state", "ranc_run_ticks", "ranc_now",
    "ranc_read_outputs", "ranc_read_potentials", "ranc_read_pending", "ranc_set_trace", "ranc_read_trace",
    "ranc_set_stream", "ranc_set_allocator", "ranc_set_option", "ranc_get_info", "ranc_comm_init",
    "ranc_gather_outputs", "ranc_comm_unique_id", "ranc_comm_init_loopback", "ranc_run_ticks_loopback",
    "ranc_plan_core_shards", "ranc_last_error", "ranc_destroy",
]

_lib = None


def load(path: str = LIB_PATH):
    """Load libranc.so (built by paper_2404_16208_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (there is no CPU fallback)")
    L = C.CDLL(path)
    st = C.c_int
    vp = C.c_void_p
    L.ranc_load_network.argtypes = [C.POINTER(NetworkDesc), C.c_int, C.POINTER(vp)]
    L.ranc_load_inputs.argtypes = [vp, C.POINTER(InputsDesc)]
    L.ranc_reset_state.argtypes = [vp]
    L.ranc_run_ticks.argtypes = [vp, C.c_int64]
    L.ranc_now.argtypes = [vp, C.POINTER(C.c_int64)]
    L.ranc_read_outputs.argtypes = [vp, vp, C.c_size_t]
    L.ranc_read_potentials.argtypes = [vp, vp, C.c_size_t]
    L.ranc_read_pending.argtypes = [vp, vp, C.c_size_t]
    L.ranc_set_trace.argtypes = [vp, C.c_uint32]
    L.ranc_read_trace.argtypes = [vp, C.c_uint32, vp, C.c_size_t, C.POINTER(C.c_size_t)]
    L.ranc_set_stream.argtypes = [vp, vp]
    L.ranc_set_allocator.argtypes = [vp, ALLOC_FN, FREE_FN, vp]
    L.ranc_set_option.argtypes = [vp, C.c_int, C.c_int64]
    L.ranc_get_info.argtypes = [vp, C.POINTER(Info)]
    L.ranc_comm_init.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int]
    L.ranc_gather_outputs.argtypes = [vp, vp, C.c_size_t, C.c_int]
    L.ranc_comm_unique_id.argtypes = [vp]
    L.ranc_comm_init_loopback.argtypes = [C.POINTER(vp), C.c_int, C.c_int]
    L.ranc_run_ticks_loopback.argtypes = [C.POINTER(vp), C.c_int, C.c_int64]
    i32p = C.POINTER(C.c_int32)
    L.ranc_plan_core_shards.argtypes = [C.POINTER(NetworkDesc), C.c_int, C.c_int, i32p, i32p, i32p, i32p, i32p,
                                        C.c_size_t, i32p, C.c_size_t]
    L.ranc_last_error.argtypes = [vp]
    L.ranc_last_error.restype = C.c_char_p
    L.ranc_destroy.argtypes = [vp]
    L.ranc_destroy.restype = None
    for f in EXPORTS:
        if f not in ("ranc_last_error", "ranc_destroy"):
            getattr(L, f).restype = st
    _lib = L
    return L
