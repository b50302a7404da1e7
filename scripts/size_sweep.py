#!/usr/bin/env python3
"""Device-resident ms per call of each kernel family over a size x radius grid
(uniform noise, L=20 unless given): the planner's crossover data.
usage: python scripts/size_sweep.py [--levels 20] [--kernels 1,2,4]"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc

ap = argparse.ArgumentParser()
ap.add_argument("--levels", type=int, default=20)
ap.add_argument("--kernels", default="1,2,4")
ap.add_argument("--sizes", default="640x480,1280x720,1920x1080,2560x1600,3840x2160,4096x4096")
ap.add_argument("--radii", default="1,2,3,5,7")
args = ap.parse_args()
s = torch.cuda.Stream()
for size in args.sizes.split(","):
    W, H = map(int, size.split("x"))
    img = torch.from_numpy(np.random.default_rng(1).integers(0, 256, (H, W, 3), dtype=np.uint8)).cuda()
    out = torch.empty_like(img)
    for r in map(int, args.radii.split(",")):
        row = [f"{size} r={r}"]
        for k in map(int, args.kernels.split(",")):
            c = opc.CudaConfig(device=0, stream=s.cuda_stream, kernel=k)
            p = opc.FilterParams(r, args.levels)
            try:
                for _ in range(2):
                    opc.apply_cuda_device(img.data_ptr(), out.data_ptr(), W, H, p, c)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    e0.record(s)
                    for _ in range(10):
                        opc.apply_cuda_device(img.data_ptr(), out.data_ptr(), W, H, p, c)
                    e1.record(s)
                s.synchronize()
                row.append(f"k{k}={e0.elapsed_time(e1) / 10:.4f}")
            except Exception as ex:  # unsupported family for these params
                row.append(f"k{k}=NA")
        print(" ".join(row), flush=True)
