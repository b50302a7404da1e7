"""The five BASELINE.json configurations as plain data.

This module imports nothing from the package and loads no library: bench.py's
reference arm reads it by file path, so the reference arm never maps the
product library (liboilpaint_b200.so).  Pattern kinds are the numbers of
include/oilpaint_b200_patterns.h (0 NOISE = the reference Noise{seed},
10 SMOOTH, 11 RECTS, 12 VIDEO = the config 2/3/5 harness generators).
"""
from __future__ import annotations

from dataclasses import dataclass

PATTERN_NOISE, PATTERN_SMOOTH, PATTERN_RECTS, PATTERN_VIDEO = 0, 10, 11, 12


@dataclass(frozen=True)
class Workload:
    name: str
    width: int
    height: int
    frames: int
    radius: int
    levels: int
    pattern: int
    seed: int
    description: str

    @property
    def megapixels(self) -> float:
        return self.frames * self.width * self.height / 1e6


# border CopyInput for all five (BASELINE.json leaves it unspecified; the
# reference default, proj/include/oilpaint/filter.hpp:21)
WORKLOADS = {
    "c1": Workload("c1", 640, 480, 1, 2, 20, PATTERN_NOISE, 1,
                   "640x480 uniform noise, r=2, L=20"),
    "c2": Workload("c2", 1920, 1080, 1, 5, 20, PATTERN_SMOOTH, 2,
                   "1920x1080 smooth sinusoids + U{-8..8}, r=5, L=20"),
    "c3": Workload("c3", 4096, 4096, 1, 10, 256, PATTERN_RECTS, 3,
                   "4096x4096 64 rectangles, r=10, L=256"),
    "c4": Workload("c4", 16384, 16384, 1, 15, 20, PATTERN_NOISE, 4,
                   "16384x16384 uniform noise, r=15, L=20"),
    "c5": Workload("c5", 3840, 2160, 64, 7, 30, PATTERN_VIDEO, 5,
                   "64 x 3840x2160 smooth field + N(0,12^2), r=7, L=30"),
}
