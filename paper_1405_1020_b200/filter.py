"""Python mirror of the reference filter interface over the C-ABI.

Reference interface (arxiv/paper_1405_1020 "oilbench", /root/reference/proj):
  enum class BorderPolicy { CopyInput, ZeroFill }       include/oilpaint/filter.hpp:13-16
  struct FilterParams { radius = 2; intensity_levels = 20;
                        border = CopyInput; }            include/oilpaint/filter.hpp:18-22
  void validate(const Image&, const FilterParams&)       src/filter.cpp:8-26
  Image apply_sequential(const Image&, const FilterParams&)   src/filter.cpp:51-68
  Image apply_parallel(const Image&, const FilterParams&, const ParallelConfig&)
                                                          src/parallel.cpp:110-132
Here an Image is a (height, width, 3) uint8 numpy array (the reference's
interleaved RGB8, stride 3*W, no padding).  Error behaviour follows the
reference: std::invalid_argument -> ValueError (InvalidArgument), runtime /
CUDA failures -> RuntimeError (CudaError), allocation -> MemoryError.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import LIB


class BorderPolicy(enum.IntEnum):
    CopyInput = 0
    ZeroFill = 1


@dataclass(frozen=True)
class FilterParams:
    radius: int = 2
    intensity_levels: int = 20
    border: BorderPolicy = BorderPolicy.CopyInput


@dataclass
class CudaConfig:
    """Engine configuration (the CUDA analogue of ParallelConfig, parallel.hpp:10-17)."""
    device: int = -1           # -1: current device
    devices: tuple = ()        # >1 entries: rows (or frames) split across these GPUs
    stream: Optional[int] = None   # cudaStream_t handle for device-pointer calls
    kernel: int = _lib.OPC_KERNEL_AUTO
    allow_levels_256: bool = False  # documented C-ABI extension (config 3)
    count_ops: bool = False    # measurement run: count executed primitives (op_counts())

    def to_c(self, device_pointers: bool = False) -> _lib.opc_config:
        flags = 0
        if device_pointers:
            flags |= _lib.OPC_FLAG_DEVICE_POINTERS
        if self.allow_levels_256:
            flags |= _lib.OPC_FLAG_ALLOW_LEVELS_256
        if self.count_ops:
            flags |= _lib.OPC_FLAG_COUNT_OPS
        return _lib.opc_config(self.device, flags, self.stream or 0, self.kernel, 0)


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference (validate, filter.cpp:8-26)."""


class CudaError(RuntimeError):
    """Runtime/CUDA failure (status OPC_ECUDA)."""


def _raise(status: int) -> None:
    if status == _lib.OPC_OK:
        return
    msg = LIB.opc_last_error().decode(errors="replace")
    if status == _lib.OPC_EINVAL:
        raise InvalidArgument(msg)
    if status == _lib.OPC_ENOMEM:
        raise MemoryError(msg)
    raise CudaError(msg)


def _check_image(img: np.ndarray) -> np.ndarray:
    if not isinstance(img, np.ndarray) or img.dtype != np.uint8 or img.ndim != 3 or img.shape[2] != 3:
        raise InvalidArgument("image must be a (height, width, 3) uint8 array")
    return np.ascontiguousarray(img)


def validate(img: np.ndarray, params: FilterParams, allow_levels_256: bool = False) -> None:
    """Reference validate (filter.cpp:8-26); raises InvalidArgument."""
    img = _check_image(img)
    h, w, _ = img.shape
    flags = _lib.OPC_FLAG_ALLOW_LEVELS_256 if allow_levels_256 else 0
    _raise(LIB.opc_validate(w, h, img.nbytes, params.radius, params.intensity_levels, flags))


def apply_cuda(img: np.ndarray, params: FilterParams = FilterParams(),
               cfg: Optional[CudaConfig] = None) -> np.ndarray:
    """apply_sequential / apply_parallel drop-in: returns a new filtered image."""
    img = _check_image(img)
    cfg = cfg or CudaConfig()
    h, w, _ = img.shape
    out = np.empty_like(img)
    c = cfg.to_c()
    if len(cfg.devices) > 1:
        _multi(img, out, 1, w, h, params, cfg, c)
        return out
    _raise(LIB.opc_filter_rgb8(img.ctypes.data, out.ctypes.data, w, h, params.radius,
                               params.intensity_levels, int(params.border), ctypes.byref(c)))
    return out


def _multi(src, dst, frames, w, h, params, cfg, c) -> None:
    devs = (ctypes.c_int32 * len(cfg.devices))(*cfg.devices)
    _raise(LIB.opc_filter_rgb8_multi(src.ctypes.data, dst.ctypes.data, frames, w, h,
                                     params.radius, params.intensity_levels, int(params.border),
                                     devs, len(cfg.devices), ctypes.byref(c)))


def apply_cuda_batch(frames: np.ndarray, params: FilterParams = FilterParams(),
                     cfg: Optional[CudaConfig] = None) -> np.ndarray:
    """Frame batch (F, H, W, 3) -> filtered batch (config 5)."""
    if frames.dtype != np.uint8 or frames.ndim != 4 or frames.shape[3] != 3:
        raise InvalidArgument("frames must be a (frames, height, width, 3) uint8 array")
    frames = np.ascontiguousarray(frames)
    cfg = cfg or CudaConfig()
    f, h, w, _ = frames.shape
    out = np.empty_like(frames)
    c = cfg.to_c()
    if len(cfg.devices) > 1:
        _multi(frames, out, f, w, h, params, cfg, c)
        return out
    _raise(LIB.opc_filter_rgb8_batch(frames.ctypes.data, out.ctypes.data, f, w, h, params.radius,
                                     params.intensity_levels, int(params.border), ctypes.byref(c)))
    return out


def band_input_rows(height: int, y_begin: int, y_end: int, radius: int) -> tuple[int, int]:
    """Input rows [lo, hi) a band [y_begin, y_end) needs (its r-row halos)."""
    lo = LIB.opc_band_in_row0(height, y_begin, radius)
    return lo, lo + LIB.opc_band_in_rows(height, y_begin, y_end, radius)


def apply_cuda_band(in_rows: np.ndarray, height: int, y_begin: int, y_end: int,
                    params: FilterParams = FilterParams(),
                    cfg: Optional[CudaConfig] = None) -> np.ndarray:
    """Output rows [y_begin, y_end) of a height-row image from its halo'd input rows."""
    in_rows = _check_image(in_rows)
    cfg = cfg or CudaConfig()
    rows, w, _ = in_rows.shape
    lo, hi = band_input_rows(height, y_begin, y_end, params.radius)
    if rows != hi - lo:
        raise InvalidArgument(f"band input must hold rows [{lo}, {hi}), got {rows} rows")
    out = np.empty((y_end - y_begin, w, 3), np.uint8)
    c = cfg.to_c()
    _raise(LIB.opc_filter_rgb8_band(in_rows.ctypes.data, out.ctypes.data, w, height, y_begin,
                                    y_end, params.radius, params.intensity_levels,
                                    int(params.border), ctypes.byref(c)))
    return out


def apply_cuda_device(in_ptr: int, out_ptr: int, width: int, height: int,
                      params: FilterParams, cfg: CudaConfig, frames: int = 1) -> None:
    """Device-resident call (pointers to 3*W*H*frames bytes on cfg.device),
    asynchronous on cfg.stream.  Used by bench.py's device-timed leg."""
    c = cfg.to_c(device_pointers=True)
    _raise(LIB.opc_filter_rgb8_batch(in_ptr, out_ptr, frames, width, height, params.radius,
                                     params.intensity_levels, int(params.border),
                                     ctypes.byref(c)))


def apply_cuda_band_device(in_ptr: int, out_ptr: int, width: int, height: int, y_begin: int,
                           y_end: int, params: FilterParams, cfg: CudaConfig) -> None:
    c = cfg.to_c(device_pointers=True)
    _raise(LIB.opc_filter_rgb8_band(in_ptr, out_ptr, width, height, y_begin, y_end,
                                    params.radius, params.intensity_levels, int(params.border),
                                    ctypes.byref(c)))


def band_begin(total: int, parts: int, k: int) -> int:
    """First row (or frame) of part k of `parts` equal contiguous parts of [0, total)."""
    return LIB.opc_band_begin(total, parts, k)


def synchronize(cfg: Optional[CudaConfig] = None) -> None:
    c = (cfg or CudaConfig()).to_c()
    _raise(LIB.opc_synchronize(ctypes.byref(c)))


def plan_kernel(width: int, height: int, radius: int, levels: int, frames: int = 1) -> int:
    if frames == 1:
        return LIB.opc_plan_kernel(width, height, radius, levels)
    return LIB.opc_plan_kernel_batch(width, height, radius, levels, frames)


def kernel_launches() -> int:
    return LIB.opc_kernel_launches()


def kernel_timing(enable: bool) -> None:
    """Start (and clear) or stop live CUDA-event timing of every kernel launch."""
    _raise(LIB.opc_kernel_timing(1 if enable else 0))


def kernel_timing_read(kernel_id: int) -> tuple[float, int]:
    """(total ms, launches) recorded for one kernel id (_lib.OPC_KID_*)."""
    ms = ctypes.c_double(0.0)
    n = ctypes.c_int64(0)
    _raise(LIB.opc_kernel_timing_read(kernel_id, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


OP_COUNT_NAMES = ("pixels", "steps", "updates", "bins_examined", "sum_pixels", "rescans",
                  "winner_changes", "nonflat_steps")


def op_counts(device: int = -1, reset: bool = True) -> dict:
    """Primitive counts accumulated by count_ops calls on `device` (see
    include/oilpaint_b200.h opc_op_counts)."""
    buf = (ctypes.c_uint64 * _lib.OPC_OPCOUNT_N)()
    _raise(LIB.opc_op_counts(device, buf, _lib.OPC_OPCOUNT_N, 1 if reset else 0))
    return dict(zip(OP_COUNT_NAMES, (int(v) for v in buf)))


def device_count() -> int:
    return LIB.opc_device_count()


def version() -> str:
    return LIB.opc_version().decode()
