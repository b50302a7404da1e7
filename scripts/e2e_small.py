#!/usr/bin/env python3
"""End-to-end (pinned host buffers, through the C-ABI host-pointer call) MP/s
of one config, median of 10 calls: the host pipeline's chunking of images
smaller than four 48 MB chunks.  usage: python scripts/e2e_small.py c2"""
import ctypes as ct, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1405_1020_b200 as opc
from paper_1405_1020_b200._lib import LIB

cfg = opc.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
W, H, r, L = cfg.width, cfg.height, cfg.radius, cfg.levels
hin = torch.empty((H, W, 3), dtype=torch.uint8).pin_memory()
cfg.generate(0, out=hin.numpy())
hout = torch.empty_like(hin).pin_memory()
c = opc.CudaConfig(device=0, allow_levels_256=L == 256).to_c()
ts = []
for i in range(13):
    t0 = time.perf_counter()
    assert LIB.opc_filter_rgb8_band(hin.data_ptr(), hout.data_ptr(), W, H, 0, H, r, L, 0, ct.byref(c)) == 0
    ts.append(time.perf_counter() - t0)
ts = sorted(ts[3:])
print(f"{cfg.name} e2e median {ts[len(ts)//2]*1e3:.3f} ms  {W*H/ts[len(ts)//2]/1e6:,.0f} MP/s")
