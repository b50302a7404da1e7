#!/usr/bin/env python3
"""Skew vs column family on smooth L=30 content (config 5 frames) across sizes
and radii: the planner threshold check for many bins (scripts/size_sweep.py is
the noise / L=20 counterpart)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc
s = torch.cuda.Stream()
for (W, H) in ((1280, 720), (1920, 1080), (2560, 1440), (3840, 2160)):
    img = torch.empty((H, W, 3), dtype=torch.uint8)
    opc.generate(opc.Pattern.VIDEO, W, H, seed=5, out=img.numpy())
    img = img.cuda(); out = torch.empty_like(img)
    for r in (3, 5, 7):
        row = [f"{W}x{H} r={r}"]
        for k in (2, 4):
            c = opc.CudaConfig(device=0, stream=s.cuda_stream, kernel=k)
            p = opc.FilterParams(r, 30)
            for _ in range(2): opc.apply_cuda_device(img.data_ptr(), out.data_ptr(), W, H, p, c)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(10): opc.apply_cuda_device(img.data_ptr(), out.data_ptr(), W, H, p, c)
                e1.record(s)
            s.synchronize()
            row.append(f"k{k}={e0.elapsed_time(e1)/10:.4f}")
        print(" ".join(row), flush=True)
