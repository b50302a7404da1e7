#!/usr/bin/env python3
"""Randomised parity campaign on one GPU: the CUDA path through the C-ABI vs the
C oracle (tests/oracle_lib.py), far more shapes than the test suite runs.

Each case draws an image shape (1 .. 700 wide, 1 .. 500 tall, biased to the
sizes where tiles, bands, rings and chunks end), a radius (0 .. 17), levels
(1 .. 256), a border policy, a content kind (noise, few colours = ties,
rectangles, smooth, constant, extremes) and then runs
  * the planner's choice and every kernel family that accepts the case,
  * a random row-band split reassembled (the multi-GPU unit),
  * a small batch of frames through the batch entry point,
comparing every output with the oracle bit for bit.

  python scripts/fuzz_parity.py --seconds 300 --seed 1 > profiles/r02_fuzz.log
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import oracle_lib  # noqa: E402
import paper_1405_1020_b200 as opc  # noqa: E402

AUTO, DIRECT, SKEW, SLIDE, COLUMN, PLANES = 0, 1, 2, 3, 4, 5
NAMES = {AUTO: "auto", DIRECT: "direct", SKEW: "skew", SLIDE: "slide", COLUMN: "column", PLANES: "planes"}
EDGES = [1, 2, 3, 15, 16, 17, 31, 32, 33, 47, 48, 49, 63, 64, 65, 95, 96, 97, 127, 128, 129, 159, 160,
         161, 255, 256, 257, 383, 384, 385]


def families(r: int, L: int):
    fam = [AUTO, DIRECT]
    if L + 1 <= 32 and r <= 15:
        fam.append(SKEW)
    if r <= 15:
        fam.append(SLIDE)
    if L + 1 <= 32 and r <= 7:
        fam.append(COLUMN)
    if L + 1 <= 32 and 1 <= r <= 7:
        fam.append(PLANES)
    return fam


def draw_dim(rng, hi):
    if rng.random() < 0.5:
        return int(min(hi, rng.choice(EDGES) + rng.integers(0, 3)))
    return int(rng.integers(1, hi + 1))


def content(rng, kind, h, w):
    if kind == 0:
        return rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    if kind == 1:  # few colours: ties between bins
        pal = rng.integers(0, 256, (int(rng.integers(2, 5)), 3), dtype=np.uint8)
        return pal[rng.integers(0, len(pal), (h, w))]
    if kind == 2:  # rectangles on a background
        img = np.empty((h, w, 3), np.uint8)
        img[:] = rng.integers(0, 256, 3, dtype=np.uint8)
        for _ in range(int(rng.integers(1, 12))):
            y0, y1 = sorted(rng.integers(0, h + 1, 2))
            x0, x1 = sorted(rng.integers(0, w + 1, 2))
            img[y0:y1, x0:x1] = rng.integers(0, 256, 3, dtype=np.uint8)
        return img
    if kind == 3:  # smooth ramp + small noise
        yy, xx = np.mgrid[0:h, 0:w]
        base = (xx * int(rng.integers(0, 4)) + yy * int(rng.integers(0, 4))) % 256
        img = np.stack([base, (base + 40) % 256, (255 - base)], -1).astype(np.int32)
        img += rng.integers(-6, 7, img.shape)
        return np.clip(img, 0, 255).astype(np.uint8)
    if kind == 4:
        img = np.empty((h, w, 3), np.uint8)
        img[:] = rng.integers(0, 256, 3, dtype=np.uint8)
        return img
    # extremes: only 0 and 255 (largest sums, bin L)
    return (rng.integers(0, 2, (h, w, 3)) * 255).astype(np.uint8)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-w", type=int, default=700)
    ap.add_argument("--max-h", type=int, default=500)
    ap.add_argument("--only", default="", help="restrict the runs to one kernel family (e.g. slide)")
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    t0 = time.time()
    cases = runs = 0
    per_family = {k: 0 for k in NAMES}
    bands = batches = 0
    fails = []
    while time.time() - t0 < args.seconds and len(fails) < 10:
        w, h = draw_dim(rng, args.max_w), draw_dim(rng, args.max_h)
        rmax = min(17, (min(w, h) - 1) // 2)
        r = int(rng.integers(0, rmax + 1))
        if rng.random() < 0.25:
            r = min(rmax, int(rng.choice([7, 8, 15, 16])))
        L = int(rng.choice([1, 2, 10, 20, 30, 31, 32, 100, 255, 256])) if rng.random() < 0.8 \
            else int(rng.integers(1, 257))
        border = int(rng.integers(0, 2))
        kind = int(rng.integers(0, 6))
        img = np.ascontiguousarray(content(rng, kind, h, w))
        want = oracle_lib.oracle_filter(img, r, L, border, threads=8)
        allow = L == 256
        p = opc.FilterParams(r, L, opc.BorderPolicy(border))
        tag = f"w={w} h={h} r={r} L={L} border={border} content={kind}"
        cases += 1
        fams = families(r, L)
        if args.only:
            fams = [k for k in fams if NAMES[k] == args.only]
            if not fams:
                continue
        for k in fams:
            got = opc.apply_cuda(img, p, opc.CudaConfig(kernel=k, allow_levels_256=allow))
            runs += 1
            per_family[k] += 1
            if not np.array_equal(got, want):
                fails.append(f"MISMATCH {NAMES[k]} {tag}: {int((got != want).any(-1).sum())} pixels")
        # a random row-band split (the multi-GPU unit), bands reassembled
        if h >= 2 and rng.random() < 0.5:
            n = int(rng.integers(2, min(h, 9) + 1))
            out = np.empty_like(img)
            k = int(rng.choice(fams))
            for j in range(n):
                y0, y1 = opc.band_begin(h, n, j), opc.band_begin(h, n, j + 1)
                if y1 <= y0:
                    continue
                lo, hi = opc.band_input_rows(h, y0, y1, r)
                out[y0:y1] = opc.apply_cuda_band(np.ascontiguousarray(img[lo:hi]), h, y0, y1, p,
                                                 opc.CudaConfig(kernel=k, allow_levels_256=allow))
            bands += 1
            if not np.array_equal(out, want):
                fails.append(f"MISMATCH bands n={n} {NAMES[k]} {tag}")
        # a small batch: this image plus shifted copies
        if rng.random() < 0.25 and w * h <= 120_000:
            nf = int(rng.integers(2, 6))
            fr = np.stack([np.roll(img, 7 * f, axis=1) for f in range(nf)])
            k = int(rng.choice(fams))
            got = opc.apply_cuda_batch(fr, p, opc.CudaConfig(kernel=k, allow_levels_256=allow))
            batches += 1
            for f in range(nf):
                wf = want if f == 0 else oracle_lib.oracle_filter(np.ascontiguousarray(fr[f]), r, L, border,
                                                                   threads=8)
                if not np.array_equal(got[f], wf):
                    fails.append(f"MISMATCH batch frame {f}/{nf} {NAMES[k]} {tag}")
                    break
    dt = time.time() - t0
    print(f"fuzz_parity seed={args.seed}: {cases} cases, {runs} single-image runs "
          f"({', '.join(f'{NAMES[k]} {v}' for k, v in per_family.items())}), "
          f"{bands} band splits, {batches} batches in {dt:.0f} s: "
          f"{'ALL BIT-EXACT' if not fails else str(len(fails)) + ' FAILURES'}")
    for f in fails:
        print(f)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
