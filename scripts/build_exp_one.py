#!/usr/bin/env python3
"""Experiment variants that differ in ONE source: recompile that source with
extra -D flags and link it with the in-tree objects of the others (build/obj).
usage: python scripts/build_exp_one.py skew.cu name=-DMACRO=V[,-DMACRO2=V] ...  (variants build in parallel)"""
import concurrent.futures as cf
import subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1405_1020_b200 import build as B

B.build()
src = sys.argv[1]
out = B.ROOT / "exp"
out.mkdir(exist_ok=True)

def one(spec):
    name, defs = spec.split("=", 1)
    defs = [d for d in defs.split(",") if d]
    obj = out / f"{name}_{src}.o"
    subprocess.run([B._nvcc(), *B.NVCC_FLAGS, *defs, "-c", str(B.CSRC / src), "-o", str(obj)], check=True)
    objs = [str(obj) if s == src else str(B.BUILD / (s + ".o")) for s in B.SOURCES]
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(out / f"{name}.so"), *objs, "-lpthread"], check=True)
    return out / f"{name}.so"

with cf.ThreadPoolExecutor(max_workers=6) as ex:
    for p in ex.map(one, sys.argv[2:]):
        print(p)
