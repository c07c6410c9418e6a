"""Plain containers for a RANC network and its input stream.

These are the arrays both sides of a parity check are fed (the oracle under
oracle/ and the C-ABI library under paper_2404_16208_b200/).  The layout is
that of ``ranc_network_desc`` / ``ranc_inputs_desc`` in include/ranc.h: all
row-major, core c = y*grid_w + x.  No arithmetic of the method lives here.

Field meanings: P:61-69 (section II, core components), S:35 (CSRAM record),
SURVEY.md 8(b).
"""
from __future__ import annotations

from dataclasses import dataclass, field, fields

import numpy as np

KIND_NONE, KIND_ROUTE, KIND_OUTPUT = 0, 1, 2
MODE_ABS, MODE_LIN = 0, 1


def words(bits: int) -> int:
    return (bits + 31) // 32


@dataclass
class Network:
    grid_w: int
    grid_h: int
    axons: int
    neurons: int
    num_types: int
    max_delay: int
    num_classes: int
    num_lines: int
    potential_bits: int
    weight_bits: int
    leak_bits: int
    threshold_bits: int
    reset_bits: int
    axon_type: np.ndarray          # u8  [G][A]
    input_line: np.ndarray         # i32 [G][A]
    crossbar: np.ndarray           # u32 [G][N][ceil(A/32)]
    weight: np.ndarray             # i16 [G][N][K]
    leak: np.ndarray               # i16 [G][N]
    pos_threshold: np.ndarray      # i16 [G][N]
    neg_threshold: np.ndarray      # i16 [G][N]
    reset_potential: np.ndarray    # i16 [G][N]
    initial_potential: np.ndarray  # i16 [G][N]
    reset_mode: np.ndarray         # u8  [G][N]
    dest_kind: np.ndarray          # u8  [G][N]
    dest_dx: np.ndarray            # i16 [G][N]
    dest_dy: np.ndarray            # i16 [G][N]
    dest_axon: np.ndarray          # i16 [G][N]
    dest_delay: np.ndarray         # u8  [G][N]
    out_class: np.ndarray          # u16 [G][N]
    name: str = "net"
    meta: dict = field(default_factory=dict)

    DTYPES = {
        "axon_type": np.uint8, "input_line": np.int32, "crossbar": np.uint32,
        "weight": np.int16, "leak": np.int16, "pos_threshold": np.int16,
        "neg_threshold": np.int16, "reset_potential": np.int16,
        "initial_potential": np.int16, "reset_mode": np.uint8, "dest_kind": np.uint8,
        "dest_dx": np.int16, "dest_dy": np.int16, "dest_axon": np.int16,
        "dest_delay": np.uint8, "out_class": np.uint16,
    }

    @property
    def G(self) -> int:
        return self.grid_w * self.grid_h

    def __post_init__(self):
        G, A, N, K = self.G, self.axons, self.neurons, self.num_types
        shapes = {
            "axon_type": (G, A), "input_line": (G, A), "crossbar": (G, N, words(A)),
            "weight": (G, N, K),
        }
        for f in fields(self):
            if f.name in self.DTYPES:
                arr = np.ascontiguousarray(getattr(self, f.name), dtype=self.DTYPES[f.name])
                want = shapes.get(f.name, (G, N))
                if arr.shape != want:
                    arr = arr.reshape(want)
                setattr(self, f.name, arr)

    def copy(self) -> "Network":
        kw = {}
        for f in fields(self):
            v = getattr(self, f.name)
            kw[f.name] = v.copy() if isinstance(v, (np.ndarray, dict)) else v
        return Network(**kw)

    def conn_dense(self) -> np.ndarray:
        """bool [G][N][A] view of the crossbar bits (test helper)."""
        A = self.axons
        bits = np.unpackbits(self.crossbar.view(np.uint8), bitorder="little")
        bits = bits.reshape(self.G, self.neurons, -1)[:, :, :A]
        return bits.astype(bool)

    @staticmethod
    def pack_conn(conn: np.ndarray) -> np.ndarray:
        """bool [G][N][A] -> u32 [G][N][ceil(A/32)], bit (a&31) of word a>>5."""
        G, N, A = conn.shape
        W = words(A)
        pad = np.zeros((G, N, W * 32), dtype=np.uint8)
        pad[:, :, :A] = conn
        return np.packbits(pad, axis=-1, bitorder="little").view(np.uint32).reshape(G, N, W)


@dataclass
class Inputs:
    num_samples: int
    num_input_ticks: int
    line_bits: np.ndarray          # u32 [S][T_in][ceil(I/32)]
    first_sample: int = 0
    labels: np.ndarray | None = None

    @staticmethod
    def from_dense(spk: np.ndarray, first_sample: int = 0, labels=None) -> "Inputs":
        """bool [S][T_in][I] -> packed Inputs."""
        S, T, I = spk.shape
        W = max(words(I), 1) if I > 0 else 0
        pad = np.zeros((S, T, W * 32), dtype=np.uint8)
        pad[:, :, :I] = spk
        lb = np.packbits(pad, axis=-1, bitorder="little").view(np.uint32).reshape(S, T, W)
        return Inputs(S, T, np.ascontiguousarray(lb), first_sample, labels)

    def dense(self, num_lines: int) -> np.ndarray:
        S, T = self.num_samples, self.num_input_ticks
        if num_lines == 0 or T == 0:
            return np.zeros((S, T, num_lines), dtype=bool)
        bits = np.unpackbits(self.line_bits.view(np.uint8), bitorder="little")
        return bits.reshape(S, T, -1)[:, :, :num_lines].astype(bool)

    def subset(self, idx) -> "Inputs":
        idx = np.asarray(idx)
        return Inputs(len(idx), self.num_input_ticks,
                      np.ascontiguousarray(self.line_bits[idx]), 0,
                      None if self.labels is None else self.labels[idx])

    def slice(self, lo: int, hi: int) -> "Inputs":
        return Inputs(hi - lo, self.num_input_ticks,
                      np.ascontiguousarray(self.line_bits[lo:hi]), self.first_sample + lo,
                      None if self.labels is None else self.labels[lo:hi])
