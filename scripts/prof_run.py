#!/usr/bin/env python3
"""Minimal device-resident driver for ncu captures and quick timing.

  python scripts/prof_run.py [--config c4] [--steps 2] [--kernel 0|1|2]

Generates the config input, copies it to the device once, runs the filter
`steps` times on one stream, prints per-step CUDA-event times.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1405_1020_b200 as opc  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--frames", type=int, default=0, help="limit frames of a batch config")
    ap.add_argument("--kt", action="store_true", help="also print per-kernel times (event hook)")
    args = ap.parse_args()
    cfg = opc.CONFIGS[args.config]
    frames = cfg.frames if args.frames <= 0 else min(cfg.frames, args.frames)
    host = np.empty((frames, cfg.height, cfg.width, 3), np.uint8)
    for f in range(frames):
        cfg.generate(f, out=host[f])
    dev_in = torch.from_numpy(host).cuda()
    dev_out = torch.empty_like(dev_in)
    s = torch.cuda.Stream()
    c = opc.CudaConfig(device=0, stream=s.cuda_stream, kernel=args.kernel,
                       allow_levels_256=cfg.levels == 256)
    p = opc.FilterParams(cfg.radius, cfg.levels)
    if args.kt:
        opc.kernel_timing(True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        for i in range(args.steps):
            opc.apply_cuda_device(dev_in.data_ptr(), dev_out.data_ptr(), cfg.width, cfg.height,
                                  p, c, frames=frames)
            ev[i + 1].record(s)
    s.synchronize()
    if args.kt:
        from paper_1405_1020_b200 import _lib
        for name in ("DIRECT", "SKEW", "SLIDE", "COLUMN", "PLANES", "PREPASS", "BORDER"):
            t, n = opc.kernel_timing_read(getattr(_lib, "OPC_KID_" + name))
            if n:
                print(f"  {name.lower()}: {t / n * 1e3:.1f} us x {n}")
        opc.kernel_timing(False)
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    mp = frames * cfg.width * cfg.height / 1e6
    print(f"{args.config} kernel={args.kernel} frames={frames} ms/step={ms} "
          f"MP/s={[round(mp / (m / 1e3), 1) for m in ms]}")


if __name__ == "__main__":
    main()
