#!/usr/bin/env python3
"""C4 end-to-end through the host-pointer C-ABI call: pinned vs pageable host
buffers (the C++ Image / numpy path is pageable)."""
import ctypes as ct, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1405_1020_b200 as opc
from paper_1405_1020_b200._lib import LIB

for name, frames in (("c4", 1), ("c5", 8)):
    cfg = opc.CONFIGS[name]
    W, H, r, L = cfg.width, cfg.height, cfg.radius, cfg.levels
    page_in = np.empty((frames, H, W, 3), np.uint8)
    for f in range(frames):
        cfg.generate(f, out=page_in[f])
    page_out = np.empty_like(page_in)
    pin_in = torch.from_numpy(page_in).pin_memory(); pin_out = torch.empty_like(pin_in).pin_memory()
    c = opc.CudaConfig(device=0).to_c()
    def call(i, o):
        rc = LIB.opc_filter_rgb8_batch(i, o, frames, W, H, r, L, 0, ct.byref(c))
        assert rc == 0, LIB.opc_last_error()
    for label, i, o in (("pinned", pin_in.data_ptr(), pin_out.data_ptr()),
                        ("pageable", page_in.ctypes.data, page_out.ctypes.data)):
        call(i, o)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter(); call(i, o); ts.append(time.perf_counter() - t0)
        dt = min(ts)
        print(f"{name} x{frames} {label:8s}: {dt*1e3:8.2f} ms  {frames*W*H/dt/1e6:8.0f} MP/s")
    assert np.array_equal(page_out, pin_out.numpy())
