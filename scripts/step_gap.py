#!/usr/bin/env python3
"""Where does the bench step's time beyond the kernel go?  C2 timed four ways
(L2 flushed before every step, CUDA events around the call): whole-image vs
band call, kernel-timing hook off / on, and a flush kernel that keeps the max
shared-memory carveout (no L1/shared reconfiguration before the step)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = opc.CONFIGS[name]
W, H = cfg.width, cfg.height
img = torch.from_numpy(cfg.generate(0)).cuda()
out = torch.empty_like(img)
s = torch.cuda.Stream()
p = opc.FilterParams(cfg.radius, cfg.levels)
c = opc.CudaConfig(device=0, stream=s.cuda_stream)
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")

def run(mode, hook, steps=20):
    opc.kernel_timing(hook)
    ms = []
    for i in range(steps + 3):
        with torch.cuda.stream(s):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            if mode == "whole":
                opc.apply_cuda_device(img.data_ptr(), out.data_ptr(), W, H, p, c)
            else:
                opc.apply_cuda_band_device(img.data_ptr(), out.data_ptr(), W, H, 0, H, p, c)
            b.record(s)
        s.synchronize()
        if i >= 3:
            ms.append(a.elapsed_time(b))
    opc.kernel_timing(False)
    ms.sort()
    return ms[len(ms) // 2]

for mode in ("whole", "band"):
    for hook in (False, True):
        print(f"{name} {mode:5s} hook={int(hook)} median {run(mode, hook):.4f} ms", flush=True)
