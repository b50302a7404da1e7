#!/usr/bin/env python3
"""Per-rank device time of an N-GPU split, measured on one GPU (rank k's share
alone): predicts the strong-scaling efficiency of bench.py --gpus N (no
collective on the data path, so ranks are independent and the job time is the
slowest share).  Single images split into row bands with r halo rows
(parallel.cpp:55-108 lifted to devices), batches into frame ranges.  Shares
under twice the L2 get the L2 flushed before every call, as bench.py does.
usage: python scripts/band_scaling.py [--config c4] [N ...]"""
import argparse
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("n", nargs="*", type=int)
ap.add_argument("--kt", action="store_true", help="per-kernel times of every share (event hook)")
args = ap.parse_args()
cfg = opc.CONFIGS[args.config]
W, H, F, r, L = cfg.width, cfg.height, cfg.frames, cfg.radius, cfg.levels
full = cfg.generate_all() if F > 1 else cfg.generate(0)[None]
p = opc.FilterParams(r, L)
s = torch.cuda.Stream()
c = opc.CudaConfig(device=0, stream=s.cuda_stream, allow_levels_256=L == 256)
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
base = None
for n in args.n or [1, 2, 4, 8]:
    worst = 0.0
    for k in sorted({0, n - 1, n // 2}):
        if F == 1:
            y0, y1 = opc.band_begin(H, n, k), opc.band_begin(H, n, k + 1)
            lo, hi = opc.band_input_rows(H, y0, y1, r)
            din = torch.from_numpy(np.ascontiguousarray(full[0, lo:hi])).cuda()
            dout = torch.empty((y1 - y0, W, 3), dtype=torch.uint8, device="cuda")
            call = lambda: opc.apply_cuda_band_device(din.data_ptr(), dout.data_ptr(), W, H, y0, y1, p, c)
        else:
            f0, f1 = opc.band_begin(F, n, k), opc.band_begin(F, n, k + 1)
            din = torch.from_numpy(np.ascontiguousarray(full[f0:f1])).cuda()
            dout = torch.empty_like(din)
            call = lambda: opc.apply_cuda_device(din.data_ptr(), dout.data_ptr(), W, H, p, c, frames=f1 - f0)
        small = din.numel() < 2 * 126 * 2**20
        for _ in range(2):
            call()
        ms = []
        for _ in range(10):
            with torch.cuda.stream(s):
                if small:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                call()
                e1.record(s)
            s.synchronize()
            ms.append(e0.elapsed_time(e1))
        worst = max(worst, sorted(ms)[len(ms) // 2])
        if args.kt:
            from paper_1405_1020_b200 import _lib
            opc.kernel_timing(True)
            for _ in range(5):
                call()
            s.synchronize()
            parts = []
            for name in ("SKEW", "SLIDE", "PLANES", "PREPASS", "BORDER"):
                t, cnt = opc.kernel_timing_read(getattr(_lib, "OPC_KID_" + name))
                if cnt:
                    parts.append(f"{name.lower()} {t / cnt * 1e3:.1f} us")
            opc.kernel_timing(False)
            print(f"    N={n} share {k}: {sorted(ms)[len(ms) // 2]:.4f} ms ({', '.join(parts)})", flush=True)
        del din, dout
    if base is None:
        base = worst * n
    mp = F * W * H / (worst / 1e3) / 1e6
    print(f"{args.config} N={n}: slowest share {worst:.4f} ms -> {mp:,.0f} MP/s job, "
          f"efficiency {base / (worst * n):.3f}", flush=True)
