"""ctypes binding of the C-ABI in include/oilpaint_b200.h.

The product path has exactly one implementation: the CUDA library
liboilpaint_b200.so built in-tree by build.py.  If it is missing this module
raises immediately -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("OILPAINT_B200_LIB",
                               Path(__file__).resolve().parent / "liboilpaint_b200.so"))

OPC_OK, OPC_EINVAL, OPC_ECUDA, OPC_ENOMEM = 0, 1, 2, 3
OPC_FLAG_DEVICE_POINTERS = 0x1
OPC_FLAG_ALLOW_LEVELS_256 = 0x2
OPC_FLAG_COUNT_OPS = 0x4
OPC_OPCOUNT_N = 8
OPC_KERNEL_AUTO, OPC_KERNEL_DIRECT, OPC_KERNEL_SKEW, OPC_KERNEL_SLIDE, OPC_KERNEL_COLUMN = 0, 1, 2, 3, 4
OPC_KERNEL_PLANES = 5

# Every symbol include/oilpaint_b200.h and include/oilpaint_b200_patterns.h declare.
EXPORTS = (
    "opc_validate", "opc_filter_rgb8", "opc_filter_rgb8_batch", "opc_filter_rgb8_band",
    "opc_band_in_row0", "opc_band_in_rows", "opc_last_error", "opc_version",
    "opc_kernel_launches", "opc_device_count", "opc_synchronize", "opc_plan_kernel",
    "opc_plan_kernel_batch",
    "opc_release", "opc_generate", "opc_filter_rgb8_multi", "opc_band_begin",
    "opc_generate_device", "opc_kernel_timing", "opc_kernel_timing_read", "opc_generate_rows",
    "opc_op_counts",
)


OPC_KID_DIRECT, OPC_KID_SKEW, OPC_KID_SLIDE, OPC_KID_PREPASS, OPC_KID_BORDER, OPC_KID_COLUMN = 1, 2, 3, 4, 5, 6
OPC_KID_PLANES = 7


class opc_config(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("stream", ctypes.c_void_p),
        ("kernel", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        if os.environ.get("OILPAINT_B200_AUTOBUILD", "1") == "1":
            from . import build as _build
            _build.build()
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run python paper_1405_1020_b200/build.py "
                              "(the CUDA library is the only implementation; no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    u8p = ctypes.c_void_p
    i32 = ctypes.c_int32
    cfgp = ctypes.POINTER(opc_config)
    lib.opc_validate.argtypes = [i32, i32, ctypes.c_uint64, i32, i32, ctypes.c_uint32]
    lib.opc_validate.restype = ctypes.c_int
    lib.opc_filter_rgb8.argtypes = [u8p, u8p, i32, i32, i32, i32, i32, cfgp]
    lib.opc_filter_rgb8.restype = ctypes.c_int
    lib.opc_filter_rgb8_batch.argtypes = [u8p, u8p, i32, i32, i32, i32, i32, i32, cfgp]
    lib.opc_filter_rgb8_batch.restype = ctypes.c_int
    lib.opc_filter_rgb8_band.argtypes = [u8p, u8p, i32, i32, i32, i32, i32, i32, i32, cfgp]
    lib.opc_filter_rgb8_band.restype = ctypes.c_int
    lib.opc_filter_rgb8_multi.argtypes = [u8p, u8p, i32, i32, i32, i32, i32, i32,
                                          ctypes.POINTER(ctypes.c_int32), i32, cfgp]
    lib.opc_filter_rgb8_multi.restype = ctypes.c_int
    lib.opc_band_begin.argtypes = [i32, i32, i32]
    lib.opc_band_begin.restype = i32
    lib.opc_band_in_row0.argtypes = [i32, i32, i32]
    lib.opc_band_in_row0.restype = i32
    lib.opc_band_in_rows.argtypes = [i32, i32, i32, i32]
    lib.opc_band_in_rows.restype = i32
    lib.opc_last_error.argtypes = []
    lib.opc_last_error.restype = ctypes.c_char_p
    lib.opc_version.argtypes = []
    lib.opc_version.restype = ctypes.c_char_p
    lib.opc_kernel_launches.argtypes = []
    lib.opc_kernel_launches.restype = ctypes.c_uint64
    lib.opc_device_count.argtypes = []
    lib.opc_device_count.restype = i32
    lib.opc_synchronize.argtypes = [cfgp]
    lib.opc_synchronize.restype = ctypes.c_int
    lib.opc_plan_kernel.argtypes = [i32, i32, i32, i32]
    lib.opc_plan_kernel.restype = i32
    lib.opc_plan_kernel_batch.argtypes = [i32, i32, i32, i32, i32]
    lib.opc_plan_kernel_batch.restype = i32
    lib.opc_release.argtypes = []
    lib.opc_release.restype = None
    lib.opc_generate.argtypes = [i32, ctypes.c_uint64, i32, i32, i32, u8p, i32]
    lib.opc_generate.restype = ctypes.c_int
    lib.opc_generate_rows.argtypes = [i32, ctypes.c_uint64, i32, i32, i32, i32, i32, u8p, i32]
    lib.opc_generate_rows.restype = ctypes.c_int
    lib.opc_generate_device.argtypes = [i32, ctypes.c_uint64, i32, i32, u8p, i32, ctypes.c_void_p]
    lib.opc_generate_device.restype = ctypes.c_int
    lib.opc_op_counts.argtypes = [i32, ctypes.POINTER(ctypes.c_uint64), i32, i32]
    lib.opc_op_counts.restype = ctypes.c_int
    lib.opc_kernel_timing.argtypes = [i32]
    lib.opc_kernel_timing.restype = ctypes.c_int
    lib.opc_kernel_timing_read.argtypes = [i32, ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_int64)]
    lib.opc_kernel_timing_read.restype = ctypes.c_int
    return lib


LIB = _load()
