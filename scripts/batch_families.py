#!/usr/bin/env python3
"""Skew vs bit-plane family on 64-frame 3840x2160 batches (r = 7, L = 30):
config 5's smooth frames and uniform noise.  Device-resident ms per batch."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc

cfg = opc.CONFIGS["c5"]
F, W, H = cfg.frames, cfg.width, cfg.height
smooth = torch.from_numpy(np.stack([cfg.generate(f) for f in range(F)])).cuda()
noise = torch.randint(0, 256, smooth.shape, dtype=torch.uint8, device="cuda")
out = torch.empty_like(smooth)
s = torch.cuda.Stream()
p = opc.FilterParams(cfg.radius, cfg.levels)
for name, src in (("smooth", smooth), ("noise", noise)):
    for k in (2, 5):
        c = opc.CudaConfig(device=0, stream=s.cuda_stream, kernel=k)
        for _ in range(2):
            opc.apply_cuda_device(src.data_ptr(), out.data_ptr(), W, H, p, c, frames=F)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(5):
                opc.apply_cuda_device(src.data_ptr(), out.data_ptr(), W, H, p, c, frames=F)
            e1.record(s)
        s.synchronize()
        print(f"{name} kernel={k} {e0.elapsed_time(e1) / 5:.3f} ms / 64 frames", flush=True)
