"""Deterministic synthetic inputs (include/oilpaint_b200_patterns.h).

Kinds NOISE/GRADIENT/UNIFORM/CHECKER restate the reference generator
(proj/src/pattern.cpp:19-88); SMOOTH/RECTS/VIDEO are the config 2/3/5
generators.  CONFIGS lists the five BASELINE.json configurations (workloads.py)
with their generators.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from ._lib import LIB
from .workloads import WORKLOADS, Workload


class Pattern(enum.IntEnum):
    NOISE = 0
    GRADIENT = 1
    UNIFORM = 2
    CHECKER = 3
    SMOOTH = 10
    RECTS = 11
    VIDEO = 12


def generate(kind: Pattern, width: int, height: int, seed: int = 0, frame: int = 0,
             threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    if out is None:
        out = np.empty((height, width, 3), np.uint8)
    assert out.shape == (height, width, 3) and out.dtype == np.uint8 and out.flags.c_contiguous
    rc = LIB.opc_generate(int(kind), seed & 0xFFFFFFFFFFFFFFFF, width, height, frame,
                          out.ctypes.data, threads)
    if rc != 0:
        raise ValueError(f"invalid pattern spec kind={kind} {width}x{height} seed={seed}")
    return out


def generate_rows(kind: Pattern, width: int, height: int, row0: int, nrows: int, seed: int = 0,
                  frame: int = 0, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """Rows [row0, row0 + nrows) of generate(kind, width, height, ...)."""
    if out is None:
        out = np.empty((nrows, width, 3), np.uint8)
    assert out.shape == (nrows, width, 3) and out.dtype == np.uint8 and out.flags.c_contiguous
    rc = LIB.opc_generate_rows(int(kind), seed & 0xFFFFFFFFFFFFFFFF, width, height, frame, row0,
                               nrows, out.ctypes.data, threads)
    if rc != 0:
        raise ValueError(f"invalid pattern spec kind={kind} {width}x{height} rows "
                         f"[{row0}, {row0 + nrows}) seed={seed}")
    return out


def generate_device(kind: Pattern, width: int, height: int, d_out: int, seed: int = 0,
                    device: int = -1, stream: int | None = None, frame: int = 0) -> None:
    """Write the pattern into device memory at address `d_out` (every kind, the
    same bytes as generate(); asynchronous on `stream`)."""
    if int(kind) == 12:  # VIDEO: frame f is the field seeded seed + f
        seed = seed + frame
    rc = LIB.opc_generate_device(int(kind), seed & 0xFFFFFFFFFFFFFFFF, width, height, d_out,
                                 device, stream or None)
    if rc != 0:
        msg = LIB.opc_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


@dataclass(frozen=True)
class BenchConfig(Workload):
    """A workload (workloads.py) with generators bound to the product library."""

    @property
    def pattern_kind(self) -> Pattern:
        return Pattern(self.pattern)

    def generate(self, frame: int = 0, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        return generate(Pattern(self.pattern), self.width, self.height, self.seed, frame, threads,
                        out)

    def generate_rows(self, row0: int, nrows: int, frame: int = 0, threads: int = 0,
                      out: np.ndarray | None = None) -> np.ndarray:
        return generate_rows(Pattern(self.pattern), self.width, self.height, row0, nrows,
                             self.seed, frame, threads, out)

    def generate_all(self, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.frames, self.height, self.width, 3), np.uint8)
        for f in range(self.frames):
            self.generate(f, threads, out[f])
        return out


CONFIGS = {k: BenchConfig(**vars(w)) for k, w in WORKLOADS.items()}
