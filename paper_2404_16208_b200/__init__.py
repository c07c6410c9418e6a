"""B200-native tick-accurate RANC core update (GPU-RANC, arXiv 2404.16208).

The product is the C-ABI library libranc.so (include/ranc.h, CUDA for
sm_100a); this package is its thin Python binding.
"""
from ._lib import (OPT_KERNEL, OPT_SAMPLE_TILE, OPT_INPUT_DECODE, OPT_STREAM, OPT_RING_LAYOUT, OPT_DEBUG_FAULT, OPT_OPERAND, SHARD_CORES, SHARD_SAMPLES,  # noqa: F401
                   TRACE_OUTPUT_EVENTS, TRACE_SPIKE_RASTER, TRACE_STATE_DIGEST, RancError)
from .sim import Simulator  # noqa: F401

__all__ = ["Simulator", "RancError", "TRACE_SPIKE_RASTER", "TRACE_OUTPUT_EVENTS", "TRACE_STATE_DIGEST", "OPT_SAMPLE_TILE",
           "OPT_INPUT_DECODE", "OPT_KERNEL", "OPT_STREAM", "OPT_RING_LAYOUT", "OPT_DEBUG_FAULT", "OPT_OPERAND", "SHARD_SAMPLES", "SHARD_CORES"]
