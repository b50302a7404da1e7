#!/usr/bin/env python3
"""A/B timing of library variants (build.build_variant) on one config, each
variant in its own process, interleaved rounds; device time per step (CUDA
events), median over steps.

  python scripts/ab_time.py --config c3 --rounds 3 lib_a.so lib_b.so ...
  (a path of "default" is the in-tree library)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import sys, json
sys.path.insert(0, %r)
import numpy as np, torch
import paper_1405_1020_b200 as opc
cfg = opc.CONFIGS[%r]
frames = min(cfg.frames, %d)
host = np.stack([cfg.generate(f) for f in range(frames)])
din = torch.from_numpy(host).cuda(); dout = torch.empty_like(din)
s = torch.cuda.Stream()
c = opc.CudaConfig(device=0, stream=s.cuda_stream, allow_levels_256=cfg.levels == 256, kernel=%d)
p = opc.FilterParams(cfg.radius, cfg.levels)
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
ms = []
ref = None
for i in range(%d):
    with torch.cuda.stream(s):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        opc.apply_cuda_device(din.data_ptr(), dout.data_ptr(), cfg.width, cfg.height, p, c, frames=frames)
        b.record(s)
    s.synchronize()
    if i >= 3: ms.append(a.elapsed_time(b))
    if ref is None: ref = dout.clone()
    else: assert torch.equal(ref, dout)
ms.sort()
print(json.dumps({"median": ms[len(ms)//2], "min": ms[0], "sum": float(dout.sum(dtype=torch.int64))}))
"""


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("libs", nargs="+")
    args = ap.parse_args()
    res = {lib: [] for lib in args.libs}
    sums = {}
    for _ in range(args.rounds):
        for lib in args.libs:
            env = dict(os.environ)
            if lib != "default":
                env["OILPAINT_B200_LIB"] = str(Path(lib).resolve())
            code = CHILD % (str(ROOT), args.config, args.frames, args.kernel, args.steps + 3)
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                 text=True, timeout=600)
            if out.returncode != 0:
                print(lib, "FAILED", out.stderr[-2000:])
                continue
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res[lib].append(d["median"])
            sums[lib] = d["sum"]
    base = None
    for lib in args.libs:
        v = sorted(res[lib])
        med = v[len(v) // 2] if v else float("nan")
        base = base or med
        print(f"{args.config} {lib:40s} median {med:.4f} ms  rounds {[round(x, 4) for x in res[lib]]}  "
              f"vs first {med / base:.3f}  checksum {sums.get(lib)}")


if __name__ == "__main__":
    main()
