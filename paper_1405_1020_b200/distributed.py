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
over NVLink between GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .filter import FilterParams, apply_cuda_band, band_begin, band_input_rows


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
    return apply_cuda_band(in_rows, height, y0, y1, params)


def filter_distributed(img: Optional[np.ndarray], params: FilterParams,
                       compute_band: Optional[BandFn] = None, group=None) -> Optional[np.ndarray]:
    """Rank 0 passes the (H, W, 3) image (others pass None); rank 0 returns the
    filtered image, the others None.  compute_band defaults to the CUDA band
    call on this process's current device."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    compute_band = compute_band or _default_band
    meta = [img.shape if rank == 0 else None]
    dist.broadcast_object_list(meta, src=0, group=group)
    h, w, _ = meta[0]
    plans = row_plan(h, params.radius, world)
    use_cuda = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if use_cuda else torch.device("cpu")

    def to_t(a: np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    mine = plans[rank]
    if rank == 0:
        for p in plans[1:]:
            if p.y1 > p.y0:
                dist.send(to_t(img[p.in_lo:p.in_hi]), dst=p.rank, group=group)
        local_in = img[mine.in_lo:mine.in_hi]
    elif mine.y1 > mine.y0:
        buf = torch.empty((mine.in_hi - mine.in_lo, w, 3), dtype=torch.uint8, device=dev)
        dist.recv(buf, src=0, group=group)
        local_in = buf.cpu().numpy()
    out_band = (compute_band(np.ascontiguousarray(local_in), h, mine.y0, mine.y1, params)
                if mine.y1 > mine.y0 else None)
    if rank == 0:
        out = np.empty((h, w, 3), np.uint8)
        out[mine.y0:mine.y1] = out_band
        for p in plans[1:]:
            if p.y1 > p.y0:
                buf = torch.empty((p.y1 - p.y0, w, 3), dtype=torch.uint8, device=dev)
                dist.recv(buf, src=p.rank, group=group)
                out[p.y0:p.y1] = buf.cpu().numpy()
        return out
    if out_band is not None:
        dist.send(to_t(out_band), dst=0, group=group)
    return None
