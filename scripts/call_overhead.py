#!/usr/bin/env python3
"""Per-call cost of the device-pointer C-ABI call for small configs: host time
per call (enqueue only, N calls then one sync) vs GPU time per call (events on
a non-default stream)."""
import ctypes as ct, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1405_1020_b200 as opc
from paper_1405_1020_b200._lib import LIB

for name in ("c1", "c2"):
    cfg = opc.CONFIGS[name]
    W, H, r, L = cfg.width, cfg.height, cfg.radius, cfg.levels
    host = torch.empty((H, W, 3), dtype=torch.uint8)
    cfg.generate(0, out=host.numpy())
    din = host.cuda(); dout = torch.empty_like(din)
    s = torch.cuda.Stream()
    c = opc.CudaConfig(device=0, stream=s.cuda_stream).to_c(); c.flags |= 1
    def call():
        assert LIB.opc_filter_rgb8(din.data_ptr(), dout.data_ptr(), W, H, r, L, 0, ct.byref(c)) == 0
    for _ in range(20): call()
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n): call()
    th = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(n): call()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"{name}: host enqueue {th*1e6:.1f} us/call, GPU {e0.elapsed_time(e1)/n*1e3:.1f} us/call")
