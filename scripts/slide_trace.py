#!/usr/bin/env python3
"""Pass-level trace of the slide kernel on config 3 (needs an OPC_SLIDE_TRACE=1
build in OILPAINT_B200_LIB): per-SM busy spans, pass duration distribution and
the slowest passes."""
import ctypes as ct, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc
from paper_1405_1020_b200._lib import LIB

cfg = opc.CONFIGS["c3"]
host = cfg.generate()
din = torch.from_numpy(host).cuda(); dout = torch.empty_like(din)
s = torch.cuda.Stream()
c = opc.CudaConfig(device=0, stream=s.cuda_stream, allow_levels_256=True)
p = opc.FilterParams(cfg.radius, cfg.levels)
buf = (ct.c_ulonglong * (4 << 16))()
f = LIB.opc_debug_slide_trace
f.argtypes = [ct.c_void_p, ct.c_int]
for it in range(3):
    opc.apply_cuda_device(din.data_ptr(), dout.data_ptr(), cfg.width, cfg.height, p, c)
    s.synchronize()
    n = f(buf, 1 << 16)
t = np.frombuffer(buf, dtype=np.uint64, count=4 * n).reshape(n, 4).astype(np.int64)
sm = t[:, 0] >> 48; kb = (t[:, 0] >> 24) & 0xFFFFFF; x0 = t[:, 0] & 0xFFFFFF; x1 = t[:, 1] & 0x3FFFFFFF; stolen = (t[:, 1] >> 30) & 1
t0 = t[:, 2] - t[:, 2].min(); t1 = t[:, 3] - t[:, 2].min(); dur = t1 - t0
print(f"stolen passes {stolen.sum()}, cols {(x1 - x0)[stolen == 1].sum()}")
print(f"passes {n}, kernel span {t1.max()/1e3:.1f} us")
end_per_sm = np.array([t1[sm == k].max() for k in np.unique(sm)])
busy_per_sm = np.array([dur[sm == k].sum() for k in np.unique(sm)])
print(f"SM end times us: min {end_per_sm.min()/1e3:.1f} median {np.median(end_per_sm)/1e3:.1f} max {end_per_sm.max()/1e3:.1f}")
print(f"pass duration us: p50 {np.percentile(dur,50)/1e3:.1f} p90 {np.percentile(dur,90)/1e3:.1f} p99 {np.percentile(dur,99)/1e3:.1f} max {dur.max()/1e3:.1f}")
print(f"pass width: p50 {np.percentile(x1-x0,50)} min {(x1-x0).min()} max {(x1-x0).max()}")
order = np.argsort(-dur)[:12]
for i in order:
    print(f"  slow pass: sm {sm[i]} band {kb[i]} cols [{x0[i]},{x1[i]}) start {t0[i]/1e3:.1f} dur {dur[i]/1e3:.1f} us")
late = np.argsort(-t1)[:8]
for i in late:
    print(f"  last to end: sm {sm[i]} band {kb[i]} cols [{x0[i]},{x1[i]}) start {t0[i]/1e3:.1f} end {t1[i]/1e3:.1f} us")
# per-band total time
bt = np.bincount(kb, weights=dur)
print("band time us (top 8):", [(int(b), round(bt[b]/1e3, 1)) for b in np.argsort(-bt)[:8]], "mean", round(bt.mean()/1e3, 1))
# warp-time accounting: busy warp-time vs resident warp-time over the kernel span
span = t1.max()
nsm = len(np.unique(sm))
print(f"busy warp-time {dur.sum()/1e3:.0f} us = {dur.sum()/span:.1f} warps busy on average over the span "
      f"({nsm} SMs); cost per column-step by pass: p10 {np.percentile(dur/(x1-x0),10):.0f} ns "
      f"p50 {np.percentile(dur/(x1-x0),50):.0f} p90 {np.percentile(dur/(x1-x0),90):.0f} max {(dur/(x1-x0)).max():.0f}")
tl = np.linspace(0, span, 25)
act = [int(((t0 <= a) & (t1 > a)).sum()) for a in tl[:-1]]
print("passes in flight at 24 sample times:", act)
if len(sys.argv) > 1:  # per-pass table for offline cost-model fits
    np.savez_compressed(sys.argv[1], sm=sm, kb=kb, x0=x0, x1=x1, t0=t0, t1=t1)
if hasattr(LIB, "opc_debug_slide_sections"):
    sec = (ct.c_ulonglong * 16)()
    LIB.opc_debug_slide_sections.argtypes = [ct.c_void_p]
    LIB.opc_debug_slide_sections(sec)
    names = ["pass start", "step walk", "count updates", "winner resolution", "winner-change sums + quotient",
             "flat emission", "jumps", "column emit + flush", "phase top"]
    tot = sum(sec[:9]); print("passes with section clocks:", sec[9] / 3)
    print("section clocks over 3 launches (lane 0 of every warp), share of the instrumented time:")
    for i, nm in enumerate(names):
        print(f"  {nm:32s} {sec[i]/3/1.965e3:10.0f} us warp-time  {sec[i]/max(tot,1):6.1%}")
