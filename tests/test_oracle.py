"""Pins the CPU oracle (oracle/oilpaint_oracle.c) against the reference itself.

Sources of truth, all produced by the reference (tests/golden/make_fixtures.py):
  * gradient8_r2_l20_zero.ppm -- the reference's own golden generator
    (proj/tests/golden/make_golden.py), used by test_filter.cpp:205-211 and
    acceptance.cpp:196-218;
  * ref_cases.npz -- 296 random cases run through the unmodified reference
    library (apply_sequential / apply_parallel / oracle::filter);
  * the pinned Noise bytes of proj/tests/test_pattern.cpp:43-50;
  * the known answers of proj/tests/test_filter.cpp and SPEC.md.
When /root/reference is present the oracle is also cross-checked live against
oracle/_ref on fresh random inputs.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np
import pytest

import oracle_lib

GOLDEN = Path(__file__).resolve().parent / "golden"
PINNED_NOISE_SEED42 = [0x95, 0x6E, 0xEB, 0x2F, 0x26, 0x32, 0xD7, 0xBD, 0x03, 0xF1, 0x66, 0xB2]


def load_cases():
    z = np.load(GOLDEN / "ref_cases.npz")
    meta, ins, outs = z["meta"], z["inputs"], z["outputs"]
    off = 0
    for w, h, r, L, border, src in meta:
        n = int(w) * int(h) * 3
        yield (int(w), int(h), int(r), int(L), int(border), int(src),
               ins[off:off + n].reshape(h, w, 3), outs[off:off + n].reshape(h, w, 3))
        off += n


def ppm_payload(path: Path) -> tuple[int, int, np.ndarray]:
    data = path.read_bytes()
    parts = data.split(b"\n", 3)
    assert parts[0] == b"P6" and parts[2] == b"255"
    w, h = map(int, parts[1].split())
    return w, h, np.frombuffer(parts[3], np.uint8).reshape(h, w, 3)


def test_intensity_bin_known_answers():
    lib = oracle_lib.oracle()
    # proj/tests/test_filter.cpp:31-35 and SPEC.md intensity_bin examples
    assert lib.oracle_intensity_bin(0, 0, 0, 20) == 0
    assert lib.oracle_intensity_bin(255, 255, 255, 20) == 20
    assert lib.oracle_intensity_bin(100, 150, 200, 20) == 11
    # test_filter.cpp:52-54: the top bin is reachable only by pure white
    assert lib.oracle_intensity_bin(255, 255, 255, 1) == 1
    assert lib.oracle_intensity_bin(255, 255, 254, 255) == 254


def test_bin_formula_equivalence_exhaustive():
    """(r+g+b)*L/765 (filter.hpp:31-35) == floor(s*L/765.0) == the float form of
    oracle.cpp:33 for every s in [0,765] and L in [1,256]."""
    s = np.arange(766, dtype=np.int64)
    for L in range(1, 257):
        exact = (s * L) // 765
        assert np.array_equal(exact, np.floor(s * L / 765.0).astype(np.int64))
        assert np.array_equal(exact, ((s * L / 3.0) / 255).astype(np.int64))
        assert exact.max() == L and (exact == L).sum() == 1  # bin L: pure white only


def test_reciprocal_division_exact():
    """q = umulhi(2s, floor(2^31/c)+1) == s // c for all c <= 1023, s <= 255c:
    the quotient the skew kernel uses for the truncating average (filter.cpp:41-43)."""
    for c in range(1, 1024):
        m = (0x80000000 // c) + 1
        s = np.arange(255 * c + 1, dtype=np.uint64)
        q = ((s << np.uint64(1)) * np.uint64(m)) >> np.uint64(32)
        assert np.array_equal(q, s // np.uint64(c)), c


def test_noise_bytes_pinned():
    lib = oracle_lib.oracle()
    buf = (ctypes.c_uint8 * 12)()
    lib.oracle_noise(42, ctypes.addressof(buf), 12)
    assert list(buf) == PINNED_NOISE_SEED42  # proj/tests/test_pattern.cpp:43-50


def test_golden_ppm_reproduced_by_oracle():
    w, h, golden = ppm_payload(GOLDEN / "gradient8_r2_l20_zero.ppm")
    assert (w, h) == (8, 8) and (GOLDEN / "gradient8_r2_l20_zero.ppm").stat().st_size == 203
    img = np.empty((8, 8, 3), np.uint8)
    oracle_lib.oracle().oracle_gradient(8, 8, img.ctypes.data)
    out = oracle_lib.oracle_filter(img, 2, 20, border=1)
    assert np.array_equal(out, golden)


def test_oracle_matches_reference_fixtures():
    n = 0
    for w, h, r, L, border, src, img, want in load_cases():
        got = oracle_lib.oracle_filter(img, r, L, border)
        assert np.array_equal(got, want), (w, h, r, L, border, src)
        n += 1
    assert n == 296


def test_oracle_threads_agree():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (61, 47, 3), dtype=np.uint8)
    a = oracle_lib.oracle_filter(img, 3, 20, 0, threads=1)
    for t in (2, 3, 8):
        assert np.array_equal(a, oracle_lib.oracle_filter(img, 3, 20, 0, threads=t))


@pytest.mark.parametrize("w,h,r,L,ok", [
    (8, 8, 4, 20, False),   # 2r >= min dim (test_filter.cpp:295-296)
    (8, 8, -1, 20, False),
    (8, 8, 1, 0, False),
    (8, 8, 1, 256, False),  # L=256 rejected by the reference contract
    (1, 1, 0, 20, True),
    (8, 8, 3, 20, True),
])
def test_oracle_validate(w, h, r, L, ok):
    rc = oracle_lib.oracle().oracle_validate(w, h, w * h * 3, r, L, 255)
    assert (rc == 0) == ok


def test_spec_examples():
    # SPEC.md filter_pixel example: five (10,20,30) vs four (200,100,50), r=1, L=10
    img = np.array([[10, 20, 30]] * 5 + [[200, 100, 50]] * 4, np.uint8).reshape(3, 3, 3)
    assert oracle_lib.oracle_filter(img, 1, 10)[1, 1].tolist() == [10, 20, 30]
    # test_filter.cpp:160-190: three 240s win, averaged back to 240
    img = np.array([[240] * 3] * 3 + [[0] * 3] * 2 + [[255] * 3] * 2 + [[60] * 3] * 2,
                   np.uint8).reshape(3, 3, 3)
    assert oracle_lib.oracle_filter(img, 1, 20)[1, 1].tolist() == [240, 240, 240]


@pytest.mark.skipif(not oracle_lib.ref_available(), reason="needs /root/reference (build box)")
def test_oracle_matches_reference_live():
    ref = oracle_lib.load_ref()
    rng = np.random.default_rng(101)
    for i in range(300):
        w, h = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        r = int(rng.integers(0, min(4, (min(w, h) - 1) // 2) + 1))
        L = int(rng.choice([1, 10, 20, 31, 255]))
        b = int(rng.integers(0, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        assert np.array_equal(oracle_lib.oracle_filter(img, r, L, b),
                              oracle_lib.ref_apply(ref, img, r, L, b)), i
    img = rng.integers(0, 256, (20, 24, 3), dtype=np.uint8)
    assert np.array_equal(oracle_lib.oracle_filter(img, 2, 256, 0),
                          oracle_lib.ref_oracle_filter(ref, img, 2, 256, 0))


def test_ref_filter_band_equals_reference_rows():
    """bench.py's CPU sample (ref_filter_band: the reference engine body on a
    band's rows, wrapping only the band plus halos) writes exactly the rows the
    reference apply_parallel produces."""
    if not oracle_lib.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = oracle_lib.load_ref()
    rng = np.random.default_rng(77)
    img = rng.integers(0, 256, (90, 53, 3), dtype=np.uint8)
    for r, L, y0, y1 in ((4, 20, 4, 86), (4, 20, 30, 41), (7, 255, 7, 8), (7, 30, 60, 83)):
        want = oracle_lib.ref_apply(ref, img, r, L, 0, engine=1, workers=3)
        out = np.zeros_like(img)
        assert ref.ref_filter_band(img.ctypes.data, out.ctypes.data, 53, 90, r, L, y0, y1, 3) == 0
        assert np.array_equal(out[y0:y1, r:53 - r], want[y0:y1, r:53 - r]), (r, L, y0, y1)
        assert not out[:y0].any() and not out[y1:].any()
