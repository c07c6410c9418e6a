"""Seeded synthetic workload generators shared by the oracle and the CUDA path.

Holds no arithmetic of the RANC method."""
from .netdef import (KIND_NONE, KIND_OUTPUT, KIND_ROUTE, MODE_ABS, MODE_LIN,  # noqa: F401
                     Inputs, Network, words)
from .rng import SplitMix64, substream  # noqa: F401
