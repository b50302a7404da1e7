"""One-process-per-GPU partition of the filter.

Every output pixel depends only on its window, so the path shards without any
data-path collective:
  * a single image is split into contiguous row bands [band_begin(H,N,k),
    band_begin(H,N,k+1)); rank k needs input rows [y0 - r, y1 + r) (the r-row
    halo is duplicated, not exchanged) -- the reference's row-band split of
    parallel_for_rows (proj/src/parallel.cpp:55-108) lifted to GPUs;
  * a frame batch is split by frame.
bench.py runs this partition with each rank generating its own share of the
deterministic input.  filter_distributed() below is the library form for a
caller that holds the image on rank 0: point-to-point scatter of the halo'd
bands, local filter, point-to-point gather (torch.distributed send/recv, NCCL
over NVLink between GPUs with the bands kept in device memory, gloo in the CPU
tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .filter import (CudaConfig, FilterParams, apply_cuda_band, apply_cuda_band_device,
                     band_begin, band_input_rows)


@dataclass(frozen=True)
class BandPlan:
    rank: int
    y0: int      # first output row of the band
    y1: int      # one past the last output row
    in_lo: int   # first input row needed (y0 - r, clipped)
    in_hi: int   # one past the last input row needed (y1 + r, clipped)


def row_plan(height: int, radius: int, world: int) -> list[BandPlan]:
    """Contiguous disjoint bands covering [0, height), with their halo'd input."""
    plans = []
    for k in range(world):
        y0, y1 = band_begin(height, world, k), band_begin(height, world, k + 1)
        lo, hi = band_input_rows(height, y0, y1, radius) if y1 > y0 else (y0, y0)
        plans.append(BandPlan(k, y0, y1, lo, hi))
    return plans


def frame_plan(frames: int, world: int) -> list[tuple[int, int]]:
    return [(band_begin(frames, world, k), band_begin(frames, world, k + 1)) for k in range(world)]


BandFn = Callable[[np.ndarray, int, int, int, FilterParams], np.ndarray]


def _default_band(in_rows, height, y0, y1, params):
    return apply_cuda_band(in_rows, height, y0, y1, params,
                           CudaConfig(allow_levels_256=params.intensity_levels == 256))


def _device_band(dev_in, height: int, y0: int, y1: int, params: FilterParams):
    """Band filter on device-resident rows (a torch uint8 CUDA tensor holding
    the halo'd input rows): the output rows stay on the device.  The library
    call runs on a side stream ordered after torch's current stream (which
    wrote dev_in) and before it (which the NCCL send that follows uses); the
    legacy default stream has no handle to pass to the C-ABI (a NULL stream
    there means the library's own stream)."""
    import torch

    rows, w, _ = dev_in.shape
    cur = torch.cuda.current_stream(dev_in.device)
    side = torch.cuda.Stream(device=dev_in.device)
    side.wait_stream(cur)
    out = torch.empty((y1 - y0, w, 3), dtype=torch.uint8, device=dev_in.device)
    cfg = CudaConfig(device=dev_in.device.index, stream=side.cuda_stream,
                     allow_levels_256=params.intensity_levels == 256)
    apply_cuda_band_device(dev_in.data_ptr(), out.data_ptr(), w, height, y0, y1, params, cfg)
    dev_in.record_stream(side)
    out.record_stream(side)
    cur.wait_stream(side)
    return out


def filter_distributed(img: Optional[np.ndarray], params: FilterParams,
                       compute_band: Optional[BandFn] = None, group=None) -> Optional[np.ndarray]:
    """Rank 0 passes the (H, W, 3) image (others pass None); rank 0 returns the
    filtered image, the others None.

    NCCL (one process per GPU) with the default band function: rank 0 uploads
    each rank's halo'd band once and sends it device to device; every rank
    filters its band in device memory (opc_filter_rgb8_band with device
    pointers) and sends the output rows back device to device; rank 0 copies
    the assembled image to the host once.  No band crosses PCIe more than
    twice (up at rank 0, down at rank 0).  With a compute_band (host arrays in
    and out, e.g. the CPU oracle in the gloo tests) the bands travel as CPU
    tensors."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    meta = [img.shape if rank == 0 else None]
    dist.broadcast_object_list(meta, src=0, group=group)
    h, w, _ = meta[0]
    plans = row_plan(h, params.radius, world)
    mine = plans[rank]
    on_device = dist.get_backend(group) == "nccl" and compute_band is None
    if not on_device:
        compute_band = compute_band or _default_band
        dev = torch.device("cpu")
    else:
        dev = torch.device("cuda", torch.cuda.current_device())

    def to_t(a: np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    if rank == 0:
        for p in plans[1:]:
            if p.y1 > p.y0:
                dist.send(to_t(img[p.in_lo:p.in_hi]), dst=p.rank, group=group)
        local_in = to_t(img[mine.in_lo:mine.in_hi]) if on_device else img[mine.in_lo:mine.in_hi]
    elif mine.y1 > mine.y0:
        local_in = torch.empty((mine.in_hi - mine.in_lo, w, 3), dtype=torch.uint8, device=dev)
        dist.recv(local_in, src=0, group=group)
        if not on_device:
            local_in = local_in.numpy()
    out_band = None
    if mine.y1 > mine.y0:
        if on_device:
            out_band = _device_band(local_in, h, mine.y0, mine.y1, params)
        else:
            out_band = to_t(compute_band(np.ascontiguousarray(local_in), h, mine.y0, mine.y1,
                                         params))
    if rank == 0:
        full = torch.empty((h, w, 3), dtype=torch.uint8, device=dev)
        full[mine.y0:mine.y1] = out_band
        for p in plans[1:]:
            if p.y1 > p.y0:
                dist.recv(full[p.y0:p.y1], src=p.rank, group=group)
        return full.cpu().numpy()
    if out_band is not None:
        dist.send(out_band, dst=0, group=group)
    return None
