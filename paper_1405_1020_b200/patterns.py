"""Deterministic synthetic inputs (include/oilpaint_b200_patterns.h).

Kinds NOISE/GRADIENT/UNIFORM/CHECKER restate the reference generator
(proj/src/pattern.cpp:19-88); SMOOTH/RECTS/VIDEO are the config 2/3/5
generators.  CONFIGS lists the five BASELINE.json configurations.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from ._lib import LIB


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
class BenchConfig:
    name: str
    width: int
    height: int
    frames: int
    radius: int
    levels: int
    pattern: Pattern
    seed: int
    description: str

    @property
    def megapixels(self) -> float:
        return self.frames * self.width * self.height / 1e6

    def generate(self, frame: int = 0, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        return generate(self.pattern, self.width, self.height, self.seed, frame, threads, out)

    def generate_all(self, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.frames, self.height, self.width, 3), np.uint8)
        for f in range(self.frames):
            self.generate(f, threads, out[f])
        return out


# BASELINE.json "configs", border CopyInput.
CONFIGS = {
    "c1": BenchConfig("c1", 640, 480, 1, 2, 20, Pattern.NOISE, 1,
                      "640x480 uniform noise, r=2, L=20"),
    "c2": BenchConfig("c2", 1920, 1080, 1, 5, 20, Pattern.SMOOTH, 2,
                      "1920x1080 smooth sinusoids + U{-8..8}, r=5, L=20"),
    "c3": BenchConfig("c3", 4096, 4096, 1, 10, 256, Pattern.RECTS, 3,
                      "4096x4096 64 rectangles, r=10, L=256"),
    "c4": BenchConfig("c4", 16384, 16384, 1, 15, 20, Pattern.NOISE, 4,
                      "16384x16384 uniform noise, r=15, L=20"),
    "c5": BenchConfig("c5", 3840, 2160, 64, 7, 30, Pattern.VIDEO, 5,
                      "64 x 3840x2160 smooth field + N(0,12^2), r=7, L=30"),
}
