#!/usr/bin/env python3
"""Executed-primitive counts of one filter launch (OPC_FLAG_COUNT_OPS) and the
per-step device time of the uncounted launch, for a BASELINE config.

  python scripts/op_counts.py [--config c3] [--steps 10]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1405_1020_b200 as opc  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--kernel", type=int, default=0)
    args = ap.parse_args()
    cfg = opc.CONFIGS[args.config]
    frames = 1 if cfg.frames == 1 else 2
    host = np.stack([cfg.generate(f) for f in range(frames)])
    dev_in = torch.from_numpy(host).cuda()
    dev_out = torch.empty_like(dev_in)
    s = torch.cuda.Stream()
    p = opc.FilterParams(cfg.radius, cfg.levels)
    base = dict(device=0, stream=s.cuda_stream, kernel=args.kernel, allow_levels_256=cfg.levels == 256)
    counted = opc.CudaConfig(count_ops=True, **base)
    plain = opc.CudaConfig(**base)
    opc.op_counts(0, reset=True)
    opc.apply_cuda_device(dev_in.data_ptr(), dev_out.data_ptr(), cfg.width, cfg.height, p, counted,
                          frames=frames)
    counts = opc.op_counts(0, reset=True)
    ref = dev_out.clone()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        for i in range(args.steps):
            opc.apply_cuda_device(dev_in.data_ptr(), dev_out.data_ptr(), cfg.width, cfg.height, p,
                                  plain, frames=frames)
            ev[i + 1].record(s)
    s.synchronize()
    assert torch.equal(ref, dev_out), "counted and plain launches differ"
    ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps))
    print(json.dumps({"config": args.config, "frames": frames, "counts": counts,
                      "ms_median": ms[len(ms) // 2], "ms_min": ms[0]}))


if __name__ == "__main__":
    main()
