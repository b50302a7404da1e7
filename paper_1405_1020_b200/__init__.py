"""oilpaint-b200: B200-native (sm_100a) histogram oil-paint filter.

A drop-in for the reference engines apply_sequential / apply_parallel of
arxiv/paper_1405_1020 ("oilbench"): the hot path is hand-written CUDA behind the
C-ABI in include/oilpaint_b200.h; this package is the thin Python host mirror
used by the tests and bench.py.
"""
from .filter import (BorderPolicy, CudaConfig, CudaError, FilterParams, InvalidArgument,
                     apply_cuda, apply_cuda_band, apply_cuda_band_device, apply_cuda_batch,
                     apply_cuda_device, band_begin, band_input_rows, device_count, kernel_launches,
                     kernel_timing, kernel_timing_read, op_counts,
                     plan_kernel, synchronize, validate, version)
from .patterns import CONFIGS, BenchConfig, Pattern, generate, generate_device, generate_rows

__all__ = [
    "BorderPolicy", "CudaConfig", "CudaError", "FilterParams", "InvalidArgument", "apply_cuda",
    "apply_cuda_band", "apply_cuda_band_device", "band_begin", "apply_cuda_batch", "apply_cuda_device",
    "band_input_rows", "device_count", "kernel_launches", "kernel_timing", "op_counts", "kernel_timing_read", "plan_kernel", "synchronize",
    "validate", "version", "CONFIGS", "BenchConfig", "Pattern", "generate", "generate_device",
    "generate_rows",
]
