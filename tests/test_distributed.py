"""CPU tests of the multi-GPU partition, world_size 2 on gloo.

The partition logic and the scatter/gather plumbing are host code; here the
per-rank compute is the CPU oracle restricted to the band (a test stand-in for
the CUDA band call), so the test runs without a GPU and checks that bands with
duplicated r-row halos reassemble the whole-image result byte for byte, with
every output row produced exactly once (the proj/tests/test_parallel.cpp:65-103
canary, lifted to ranks).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle_lib
from paper_1405_1020_b200 import FilterParams
from paper_1405_1020_b200.distributed import filter_distributed, frame_plan, row_plan


def oracle_band(in_rows, height, y0, y1, params):
    """Output rows [y0, y1) from halo'd input rows, via the oracle on the sub-image."""
    r = params.radius
    lo = max(0, y0 - r)
    sub = oracle_lib.oracle_filter(in_rows, r, params.intensity_levels, int(params.border))
    out = sub[y0 - lo:y1 - lo].copy()
    # rows that are interior in the full image but border in the sub-image
    for y in range(y0, y1):
        interior = r <= y < height - r
        local_interior = r <= (y - lo) < in_rows.shape[0] - r
        if interior and not local_interior:
            raise AssertionError("band input lacks halo rows")
        if not interior:
            out[y - y0] = in_rows[y - lo] if params.border == 0 else 0
    return out


@pytest.mark.parametrize("h,r,world", [(50, 3, 2), (7, 3, 2), (64, 15, 8), (301, 15, 3), (5, 0, 8)])
def test_row_plan_covers_rows_exactly_once(h, r, world):
    plans = row_plan(h, r, world)
    hits = np.zeros(h, int)
    for p in plans:
        hits[p.y0:p.y1] += 1
        assert p.in_lo == max(0, p.y0 - r) and p.in_hi == min(h, p.y1 + r) or p.y1 == p.y0
    assert (hits == 1).all()


def test_frame_plan():
    for frames, world in ((64, 1), (64, 8), (64, 3), (5, 8)):
        parts = frame_plan(frames, world)
        assert sum(e - b for b, e in parts) == frames
        assert all(parts[k][1] == parts[k + 1][0] for k in range(world - 1))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, img, params, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = filter_distributed(img if rank == 0 else None, params, compute_band=oracle_band)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,r,L,border", [(2, 3, 20, 0), (2, 15, 20, 1), (3, 2, 255, 0)])
def test_gloo_band_scatter_gather_matches_whole_image(world, r, L, border):
    rng = np.random.default_rng(world * 100 + r)
    img = rng.integers(0, 256, (97, 61, 3), dtype=np.uint8)
    params = FilterParams(r, L, border)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, img, params, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle_lib.oracle_filter(img, r, L, border)
    assert np.array_equal(res, want)


def _nccl_worker(port, img, params, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        q.put(filter_distributed(img, params))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_device_band_path(gpu):
    """The NCCL form keeps bands in device memory (opc_filter_rgb8_band with
    device pointers on torch's stream); world size 1 on the one GPU a test box
    has, checked against the oracle (L = 256 exercises the extension flag)."""
    rng = np.random.default_rng(17)
    img = rng.integers(0, 256, (203, 157, 3), dtype=np.uint8)
    for params in (FilterParams(6, 20, 0), FilterParams(4, 256, 1)):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=_nccl_worker, args=(_free_port(), img, params, q))
        p.start()
        res = q.get(timeout=300)
        p.join(timeout=60)
        assert p.exitcode == 0
        want = oracle_lib.oracle_filter(img, params.radius, params.intensity_levels,
                                        int(params.border))
        assert np.array_equal(res, want)
