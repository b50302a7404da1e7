"""Test-side loaders of the parity checkers (TEST INFRASTRUCTURE ONLY).

  oracle/liboilpaint_oracle.so   our C restatement of the reference hot path
  oracle/_ref/libref_oilpaint.so the unmodified reference library (+ our shim),
                                 built from /root/reference/proj by oracle/Makefile

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use these.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"
ORACLE_SO = ORACLE_DIR / "liboilpaint_oracle.so"
REF_SO = ORACLE_DIR / "_ref" / "libref_oilpaint.so"


def _make() -> None:
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True, capture_output=True)


def load_oracle() -> ctypes.CDLL:
    if not ORACLE_SO.exists():
        _make()
    lib = ctypes.CDLL(str(ORACLE_SO))
    vp, i32 = ctypes.c_void_p, ctypes.c_int
    lib.oracle_intensity_bin.argtypes = [ctypes.c_uint8] * 3 + [i32]
    lib.oracle_intensity_bin.restype = i32
    lib.oracle_validate.argtypes = [i32, i32, ctypes.c_uint64, i32, i32, i32]
    lib.oracle_validate.restype = i32
    lib.oracle_filter.argtypes = [vp, vp, i32, i32, i32, i32, i32]
    lib.oracle_filter.restype = i32
    lib.oracle_filter_mt.argtypes = [vp, vp, i32, i32, i32, i32, i32, i32]
    lib.oracle_filter_mt.restype = i32
    lib.oracle_noise.argtypes = [ctypes.c_uint64, vp, ctypes.c_uint64]
    lib.oracle_noise.restype = None
    lib.oracle_gradient.argtypes = [i32, i32, vp]
    lib.oracle_gradient.restype = None
    return lib


def ref_available() -> bool:
    if REF_SO.exists():
        return True
    if Path("/root/reference/proj/src/filter.cpp").exists():
        _make()
    return REF_SO.exists()


def load_ref() -> ctypes.CDLL:
    if not ref_available():
        raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
    lib = ctypes.CDLL(str(REF_SO))
    vp, i32 = ctypes.c_void_p, ctypes.c_int
    lib.ref_last_error.restype = ctypes.c_char_p
    lib.ref_hardware_concurrency.restype = ctypes.c_uint
    lib.ref_apply.argtypes = [vp, vp, i32, i32, i32, i32, i32, i32, i32]
    lib.ref_apply.restype = i32
    lib.ref_oracle_filter.argtypes = [vp, vp, i32, i32, i32, i32, i32]
    lib.ref_oracle_filter.restype = i32
    lib.ref_filter_rows_any_levels.argtypes = [vp, vp, i32, i32, i32, i32, i32, i32]
    lib.ref_filter_rows_any_levels.restype = i32
    lib.ref_filter_band.argtypes = [vp, vp, i32, i32, i32, i32, i32, i32, i32]
    lib.ref_filter_band.restype = i32
    lib.ref_generate.argtypes = [i32, ctypes.c_uint64, i32, i32, vp]
    lib.ref_generate.restype = i32
    lib.ref_harness_generate_rows.argtypes = [i32, ctypes.c_uint64, i32, i32, i32, i32, i32, vp,
                                              i32]
    lib.ref_harness_generate_rows.restype = i32
    lib.ref_write_ppm.argtypes = [vp, i32, i32, vp, ctypes.c_long]
    lib.ref_write_ppm.restype = ctypes.c_long
    return lib


_ORACLE = None


def oracle() -> ctypes.CDLL:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = load_oracle()
    return _ORACLE


def oracle_filter(img: np.ndarray, radius: int, levels: int, border: int = 0,
                  threads: int = 1) -> np.ndarray:
    """CPU restatement (oracle/oilpaint_oracle.c) of apply_sequential."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w, _ = img.shape
    out = np.empty_like(img)
    lib = oracle()
    if threads > 1:
        rc = lib.oracle_filter_mt(img.ctypes.data, out.ctypes.data, w, h, radius, levels, border,
                                  threads)
    else:
        rc = lib.oracle_filter(img.ctypes.data, out.ctypes.data, w, h, radius, levels, border)
    if rc != 0:
        raise ValueError(f"oracle rejected {w}x{h} r={radius} L={levels}")
    return out


def ref_apply(lib: ctypes.CDLL, img: np.ndarray, radius: int, levels: int, border: int = 0,
              engine: int = 0, workers: int = 0) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w, _ = img.shape
    out = np.empty_like(img)
    rc = lib.ref_apply(img.ctypes.data, out.ctypes.data, w, h, radius, levels, border, engine,
                       workers)
    if rc == 1:
        raise ValueError(lib.ref_last_error().decode())
    if rc != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return out


def ref_oracle_filter(lib: ctypes.CDLL, img: np.ndarray, radius: int, levels: int,
                      border: int = 0) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w, _ = img.shape
    out = np.empty_like(img)
    if lib.ref_oracle_filter(img.ctypes.data, out.ctypes.data, w, h, radius, levels, border):
        raise RuntimeError(lib.ref_last_error().decode())
    return out


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
