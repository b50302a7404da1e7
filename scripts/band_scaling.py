#!/usr/bin/env python3
"""Per-rank device time of the C4 row bands of an N-GPU split, measured on one
GPU (rank k's band alone): predicts strong-scaling efficiency of bench.py
--gpus N (no collective on the data path, so ranks are independent).
usage: python scripts/band_scaling.py [N ...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc

cfg = opc.CONFIGS["c4"]
W, H, r, L = cfg.width, cfg.height, cfg.radius, cfg.levels
full = cfg.generate(0)
p = opc.FilterParams(r, L)
s = torch.cuda.Stream()
c = opc.CudaConfig(device=0, stream=s.cuda_stream)
base = None
for n in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    worst = 0.0
    for k in sorted({0, n - 1, n // 2}):
        y0, y1 = opc.band_begin(H, n, k), opc.band_begin(H, n, k + 1)
        lo, hi = opc.band_input_rows(H, y0, y1, r)
        din = torch.from_numpy(np.ascontiguousarray(full[lo:hi])).cuda()
        dout = torch.empty((y1 - y0, W, 3), dtype=torch.uint8, device="cuda")
        for _ in range(2):
            opc.apply_cuda_band_device(din.data_ptr(), dout.data_ptr(), W, H, y0, y1, p, c)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(10):
                opc.apply_cuda_band_device(din.data_ptr(), dout.data_ptr(), W, H, y0, y1, p, c)
            e1.record(s)
        s.synchronize()
        worst = max(worst, e0.elapsed_time(e1) / 10)
        del din, dout
    if base is None:
        base = worst * n
    mp = W * H / (worst / 1e3) / 1e6
    print(f"N={n}: slowest band {worst:.3f} ms -> {mp:,.0f} MP/s job, efficiency {base / (worst * n):.3f}", flush=True)
