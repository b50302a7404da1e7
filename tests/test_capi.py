"""CPU tests of the C-ABI boundary (no GPU compute).

  * liboilpaint_b200.so loads and exports every symbol include/*.h declares;
  * opc_validate mirrors the reference validate (proj/src/filter.cpp:8-26),
    including its messages and the documented L=256 extension;
  * the band helpers and kernel planner (host logic);
  * the deterministic input generators (the reference Noise stream pinned by
    proj/tests/test_pattern.cpp:43-50, Gradient, and thread-count independence);
  * without a GPU the filter call fails loudly (status OPC_ECUDA), never falls
    back to a CPU path.
"""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle_lib
import paper_1405_1020_b200 as opc
from paper_1405_1020_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols() -> set[str]:
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        names |= set(re.findall(r"\b(opc_\w+)\s*\(", h.read_text()))
    return names


def test_library_exports_every_declared_symbol():
    decl = declared_symbols()
    assert decl, "no declarations found"
    assert decl == set(_lib.EXPORTS)
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in decl:
        assert hasattr(lib, name), name


def test_product_library_does_not_link_the_oracle():
    import subprocess
    out = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "oracle" not in out and "ref_oilpaint" not in out
    syms = subprocess.run(["nm", "-D", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "oracle_" not in syms and "ref_" not in syms.replace("_ref_", "")


@pytest.mark.parametrize("w,h,r,L,flags,ok,msg", [
    (8, 8, 4, 20, 0, False, "leaves no interior for a 8x8 image"),
    (8, 8, -1, 20, 0, False, "radius must be >= 0, got -1"),
    (8, 8, 1, 0, 0, False, "intensity_levels must be in [1, 255], got 0"),
    (8, 8, 1, 256, 0, False, "intensity_levels must be in [1, 255], got 256"),
    (8, 8, 1, 256, 2, True, ""),
    (8, 8, 1, 257, 2, False, "intensity_levels must be in [1, 256], got 257"),
    (1, 1, 0, 20, 0, True, ""),
    (8, 8, 3, 20, 0, True, ""),
    (0, 4, 0, 20, 0, False, "image dimensions must be positive"),
])
def test_validate_mirrors_reference(w, h, r, L, flags, ok, msg):
    rc = _lib.LIB.opc_validate(w, h, w * h * 3, r, L, flags)
    assert (rc == 0) == ok
    if not ok:
        assert rc == _lib.OPC_EINVAL
        assert msg in _lib.LIB.opc_last_error().decode()


def test_validate_data_length():
    assert _lib.LIB.opc_validate(4, 4, 47, 1, 20, 0) == _lib.OPC_EINVAL
    assert "does not match" in _lib.LIB.opc_last_error().decode()
    with pytest.raises(opc.InvalidArgument):
        opc.validate(np.zeros((8, 8, 3), np.uint8), opc.FilterParams(4, 20))
    opc.validate(np.zeros((8, 8, 3), np.uint8), opc.FilterParams(3, 20))


@pytest.mark.skipif(not oracle_lib.ref_available(), reason="needs the reference build")
def test_validate_agrees_with_reference_on_random_params():
    ref = oracle_lib.load_ref()
    rng = np.random.default_rng(3)
    for _ in range(300):
        w, h = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        r, L = int(rng.integers(-2, 7)), int(rng.integers(-1, 259))
        img = np.zeros((h, w, 3), np.uint8)
        ours = _lib.LIB.opc_validate(w, h, w * h * 3, r, L, 0)
        out = np.empty_like(img)
        theirs = ref.ref_apply(img.ctypes.data, out.ctypes.data, w, h, r, L, 0, 0, 0)
        assert (ours == 0) == (theirs == 0), (w, h, r, L)
        if ours:
            assert _lib.LIB.opc_last_error().decode() == ref.ref_last_error().decode()


def test_band_helpers():
    L = _lib.LIB
    assert [L.opc_band_begin(100, 3, k) for k in range(4)] == [0, 33, 66, 100]
    assert L.opc_band_in_row0(100, 0, 15) == 0
    assert L.opc_band_in_row0(100, 40, 15) == 25
    assert L.opc_band_in_rows(100, 40, 60, 15) == 50
    assert L.opc_band_in_rows(100, 90, 100, 15) == 25


def test_kernel_planner():
    P = _lib.OPC_KERNEL_PLANES
    assert opc.plan_kernel(640, 480, 2, 20) == P  # r <= 7, L+1 <= 32: bit-plane family at every size
    assert opc.plan_kernel(640, 480, 0, 20) == _lib.OPC_KERNEL_COLUMN  # r = 0 (identity)
    assert opc.plan_kernel(640, 480, 2, 255) == _lib.OPC_KERNEL_DIRECT  # many bins, small r
    assert opc.plan_kernel(4000, 4000, 2, 20) == P
    assert opc.plan_kernel(1920, 1080, 5, 20) == P
    assert opc.plan_kernel(1920, 1080, 8, 20) == _lib.OPC_KERNEL_SKEW  # bit-plane family: r <= 7
    assert opc.plan_kernel(2560, 1600, 7, 20) == P
    assert opc.plan_kernel(16384, 16384, 15, 20) == _lib.OPC_KERNEL_SKEW
    assert opc.plan_kernel(3840, 2160, 7, 30) == P
    assert opc.plan_kernel(3840, 2160, 7, 30, frames=64) == _lib.OPC_KERNEL_SKEW  # video batch
    assert opc.plan_kernel(3840, 2160, 7, 30, frames=4) == P
    assert opc.plan_kernel(3840, 2160, 7, 20, frames=64) == P  # 21 bins: no bin window
    assert opc.plan_kernel(3840, 2160, 7, 31) == P  # 32 bins: one bit each in the plane words
    assert opc.plan_kernel(3840, 2160, 7, 32) == _lib.OPC_KERNEL_SLIDE  # 33 bins
    assert opc.plan_kernel(4096, 4096, 10, 256) == _lib.OPC_KERNEL_SLIDE
    assert opc.plan_kernel(300, 300, 15, 100) == _lib.OPC_KERNEL_SLIDE
    assert opc.plan_kernel(100, 100, 16, 20) == _lib.OPC_KERNEL_DIRECT
    assert opc.plan_kernel(8, 8, 4, 20) == -1


def test_noise_generator_matches_reference_stream():
    img = opc.generate(opc.Pattern.NOISE, 4, 1, seed=42)
    assert img.reshape(-1).tolist() == [0x95, 0x6E, 0xEB, 0x2F, 0x26, 0x32, 0xD7, 0xBD,
                                        0x03, 0xF1, 0x66, 0xB2]
    big = opc.generate(opc.Pattern.NOISE, 333, 97, seed=4)
    buf = np.empty(big.size, np.uint8)
    oracle_lib.oracle().oracle_noise(4, buf.ctypes.data, buf.size)
    assert np.array_equal(big.reshape(-1), buf)


def test_gradient_generator_matches_oracle():
    for w, h in ((8, 8), (1, 1), (13, 5)):
        a = opc.generate(opc.Pattern.GRADIENT, w, h)
        b = np.empty_like(a)
        oracle_lib.oracle().oracle_gradient(w, h, b.ctypes.data)
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", [opc.Pattern.NOISE, opc.Pattern.SMOOTH, opc.Pattern.RECTS,
                                  opc.Pattern.VIDEO])
def test_generators_independent_of_thread_count(kind):
    a = opc.generate(kind, 301, 157, seed=9, frame=2, threads=1)
    for t in (2, 7, 16):
        assert np.array_equal(a, opc.generate(kind, 301, 157, seed=9, frame=2, threads=t))


def test_config_generators_shape_and_content():
    c2 = opc.CONFIGS["c2"].generate()
    assert c2.shape == (1080, 1920, 3)
    # smooth: neighbouring pixels differ little (sinusoids + U{-8..8})
    assert np.abs(np.diff(c2.astype(int), axis=1)).mean() < 12
    c3 = opc.CONFIGS["c3"].generate()
    assert len(np.unique(c3.reshape(-1, 3), axis=0)) <= 65  # background + 64 rectangles
    v0, v1 = opc.CONFIGS["c5"].generate(0), opc.CONFIGS["c5"].generate(1)
    assert not np.array_equal(v0, v1)
    f = v0.astype(float)
    resid = f[:, 1:-1] - (f[:, :-2] + f[:, 2:]) / 2  # ~ N(0, 1.5 * 12^2) on the smooth field
    assert 12 < resid.std() < 18  # Gaussian sigma 12 noise present


def test_filter_without_gpu_fails_loudly():
    if opc.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(opc.CudaError, match="no CUDA device"):
        opc.apply_cuda(np.zeros((8, 8, 3), np.uint8), opc.FilterParams(1, 20))


def test_generate_device_without_gpu_fails_loudly():
    if opc.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        opc.generate_device(opc.Pattern.NOISE, 8, 8, 0)
