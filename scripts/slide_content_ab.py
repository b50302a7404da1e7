#!/usr/bin/env python3
"""Slide family on other content than config 3: device-resident kernel times of
OILPAINT_B200_LIB on noise, few-colour and smooth images (2048^2, r = 10, L = 256)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc

rng = np.random.default_rng(7)
H = W = 2048
yy, xx = np.mgrid[0:H, 0:W]
base = ((xx + 2 * yy) // 8) % 256
imgs = {
    "noise": rng.integers(0, 256, (H, W, 3), dtype=np.uint8),
    "4 colours": rng.integers(0, 256, (4, 3), dtype=np.uint8)[rng.integers(0, 4, (H, W))],
    "smooth ramp + noise": np.clip(np.stack([base, (base + 40) % 256, 255 - base], -1)
                                   + rng.integers(-6, 7, (H, W, 3)), 0, 255).astype(np.uint8),
}
p = opc.FilterParams(10, 256)
s = torch.cuda.Stream()
c = opc.CudaConfig(device=0, stream=s.cuda_stream, kernel=3, allow_levels_256=True)
for name, img in imgs.items():
    din = torch.from_numpy(np.ascontiguousarray(img)).cuda(); dout = torch.empty_like(din)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    with torch.cuda.stream(s):
        for i in range(6):
            ev[i].record(s)
            opc.apply_cuda_device(din.data_ptr(), dout.data_ptr(), W, H, p, c)
        end = torch.cuda.Event(enable_timing=True); end.record(s)
    s.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(1, 5)]
    print(f"{name:22s} {np.median(ms):8.3f} ms/launch")
