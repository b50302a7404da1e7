#!/usr/bin/env python3
"""Lane-by-lane Python model of the skew kernel schedule (debugging aid).

Executes exactly the schedule of paper_1405_1020_b200/csrc/skew.cu (virtual
columns, sheared loads, E-slot ring with per-step zeroing, staggered init,
staging/flush) on small images with unbounded Python ints instead of packed
words, and compares with the oracle.  Any schedule bug shows up here on the
CPU before a GPU run.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tests"))



def model(img: np.ndarray, r: int, L: int, segw: int | None = None) -> np.ndarray:
    h, w, _ = img.shape
    out = img.copy()
    w2 = 2 * r + 1
    nb = L + 1
    SLOTS, B = (64, 16) if w2 <= 16 else (96, 32)
    s_bins = (img.astype(np.int64).sum(2) * L) // 765
    y_lo, y_hi, x_lo, x_hi = r, h - r, r, w - r
    if y_hi <= y_lo or x_hi <= x_lo:
        return out
    y_base = y_lo - r
    nbands = (y_hi - y_lo + 31) // 32
    Hs = 32 * nbands + 64
    ndiag = w + Hs
    S = {}
    for y in range(y_base, y_base + Hs):
        for x in range(w + 32):
            S[(x + y - y_base) * Hs + (y - y_base)] = (x, y) if (x < w and y < h) else None
    iw = x_hi - x_lo
    segw = segw or iw
    nsegs = (iw + segw - 1) // segw

    def val(idx):
        if idx not in S:
            return None  # garbage
        if S[idx] is None:
            return (0, (0, 0, 0))  # zero entry (padding)
        x, y = S[idx]
        return (int(s_bins[y, x]), tuple(int(c) for c in img[y, x]))

    for kb in range(nbands):
        for js in range(nsegs):
            yb = y_lo + 32 * kb
            xs = x_lo + js * segw
            xe = min(xs + segw, x_hi)
            NV = w2 + (xe - xs)
            X0 = xs - w2
            R0 = yb - r - y_base
            D0 = xs - r + R0
            E = [dict() for _ in range(SLOTS)]
            win = [dict() for _ in range(32)]
            stage = [[None] * 32 for _ in range(32)]

            def fetch(s, t):
                v = s - t
                vi = s - t + w2
                L_ = {}
                if 0 <= v < NV:
                    L_["a"] = val((D0 + s + w2) * Hs + R0 + t + w2)
                    L_["b"] = val((D0 + s) * Hs + R0 + t)
                    if v >= w2:
                        L_["c"] = val((D0 + s) * Hs + R0 + t + w2)
                        L_["d"] = val((D0 + s - w2) * Hs + R0 + t)
                if t < w2 and 0 <= vi < NV:
                    L_["i1"] = val((D0 + s + w2) * Hs + R0 + t)  # column vi, row t
                    if vi >= w2:
                        L_["i2"] = val((D0 + s) * Hs + R0 + t)  # column vi - w2, row t (= b)
                return L_

            def add(dct, e, sign):
                assert e is not None, "garbage entry used"
                b, (R, G, B) = e
                c = dct.get(b, (0, 0, 0, 0))
                dct[b] = (c[0] + sign, c[1] + sign * R, c[2] + sign * G, c[3] + sign * B)

            nphases = ((NV - 1) >> 5) + 2
            for p in range(-1, nphases):
                for ss in range(32):
                    s = 32 * p + ss
                    cur = [fetch(s, t) for t in range(32)]
                    for t in range(32):
                        v = s - t
                        row_ok = yb + t < y_hi
                        if 0 <= v < NV:
                            slot = v % SLOTS
                            e = dict(E[slot])
                            if v >= w2 and row_ok:
                                best, bc = 0, win[t].get(0, (0,))[0]
                                for b in range(1, nb):
                                    c = win[t].get(b, (0,))[0]
                                    if c > bc:
                                        best, bc = b, c
                                cnt, sr, sg, sbb = win[t][best]
                                stage[t][v & 31] = (sr // cnt, sg // cnt, sbb // cnt)
                            for b, q in e.items():
                                c = win[t].get(b, (0, 0, 0, 0))
                                win[t][b] = tuple(x + y for x, y in zip(c, q))
                            add(E[slot], cur[t]["a"], +1)
                            add(E[slot], cur[t]["b"], -1)
                            if v >= w2:
                                add(E[slot], cur[t]["c"], -1)
                                add(E[slot], cur[t]["d"], +1)
                        vi = s - t + w2
                        if t < w2 and 0 <= vi < NV:
                            slot = vi % SLOTS
                            add(E[slot], cur[t]["i1"], +1)
                            if vi >= w2:
                                add(E[slot], cur[t]["i2"], -1)
                    fr = (s + 1) & 31
                    for lane in range(32):
                        vv = s - fr - 31 + lane
                        if w2 <= vv < NV and yb + fr < y_hi:
                            out[yb + fr, X0 + vv] = stage[fr][lane]
                    if s % B == B - 1:  # batch-clear the slots of columns s+1+w2 .. s+B+w2
                        for c in range(s + 1 + w2, s + B + w2 + 1):
                            E[c % SLOTS] = dict()
    return out


if __name__ == "__main__":
    import oracle_lib

    rng = np.random.default_rng(1)
    cases = [(14, 4, 0, 1), (20, 30, 2, 20), (40, 70, 3, 10), (33, 45, 5, 31), (50, 60, 7, 30),
             (60, 70, 8, 20), (70, 50, 15, 20)]
    for h, w, r, L in cases:
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        got = model(img, r, L, segw=int(rng.integers(5, 40)))
        want = oracle_lib.oracle_filter(img, r, L, 0)
        bad = np.argwhere((got != want).any(2))
        print(h, w, r, L, "OK" if len(bad) == 0 else f"MISMATCH at {bad[:5].tolist()}")
