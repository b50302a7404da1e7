#!/usr/bin/env python3
"""Where does the C4 end-to-end time go?  (pinned host buffers, one B200)
 a) the library's host-pointer call (H2D / kernels / D2H pipelined by capi.cu)
 b) the same row-chunk schedule as pure copies (no kernels)
 c) device-resident kernels per chunk size"""
import ctypes as ct, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc
from paper_1405_1020_b200._lib import LIB

cfg = opc.CONFIGS["c4"]
W, H, r, L = cfg.width, cfg.height, cfg.radius, cfg.levels
host_in = torch.empty((H, W, 3), dtype=torch.uint8).pin_memory()
cfg.generate(0, out=host_in.numpy())
host_out = torch.empty_like(host_in).pin_memory()
c = opc.CudaConfig(device=0).to_c()

def lib_call():
    rc = LIB.opc_filter_rgb8_band(host_in.data_ptr(), host_out.data_ptr(), W, H, 0, H, r, L, 0, ct.byref(c))
    assert rc == 0
lib_call()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); lib_call(); dt = time.perf_counter() - t0
    print(f"a) library e2e {dt*1e3:.2f} ms  {W*H/dt/1e6:.0f} MP/s")

# b) copies only, chunk schedule like capi.cu (ramp 64..512 rows, ~1024-row middle)
row = W * 3
sizes = [64, 128, 256, 512]
mid = H - 2 * sum(sizes); n = -(-mid // 1024)
sched = sizes + [mid * (k + 1) // n - mid * k // n for k in range(n)] + sizes[::-1]
d_in = torch.empty(H * row, dtype=torch.uint8, device="cuda"); d_out = torch.empty_like(d_in)
hi, ho = host_in.view(-1), host_out.view(-1)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def copies(delay_kernel_ms=0.0):
    y = 0; evs = []
    for q in sched:
        a, b = y * row, (y + q) * row
        with torch.cuda.stream(s1):
            d_in[a:b].copy_(hi[a:b], non_blocking=True); e = torch.cuda.Event(); e.record(s1)
        with torch.cuda.stream(s2):
            s2.wait_event(e); ho[a:b].copy_(d_out[a:b], non_blocking=True)
        y += q
for _ in range(2): copies()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); copies(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"b) copies only {dt*1e3:.2f} ms  ({len(sched)} chunks)")

# c) device-resident kernels per chunk of q rows (band in the middle of the image)
dev_in = host_in.cuda(); dev_out = torch.empty_like(dev_in)
cd = opc.CudaConfig(device=0, stream=torch.cuda.current_stream().cuda_stream).to_c(); cd.flags |= 1
for q in (64, 256, 512, 1024, 2048, H):
    y0 = max(0, H // 2 - q // 2) if q < H else 0
    lo = LIB.opc_band_in_row0(H, y0, r)
    def run():
        rc = LIB.opc_filter_rgb8_band(dev_in.data_ptr() + lo * row, dev_out.data_ptr() + y0 * row, W, H, y0, y0 + q, r, L, 0, ct.byref(cd))
        assert rc == 0
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [run() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"c) kernels for {q:5d} rows: {ms:.3f} ms  ({ms / q * H:.2f} ms per full image)")
