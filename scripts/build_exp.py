#!/usr/bin/env python3
"""Build experiment variants of the product library into exp/<name>.so.
usage: python scripts/build_exp.py name=-DMACRO=V[,-DMACRO2=V] ..."""
import subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1405_1020_b200 import build as B

out = B.ROOT / "exp"
out.mkdir(exist_ok=True)
for spec in sys.argv[1:]:
    name, defs = spec.split("=", 1)
    defs = [d for d in defs.split(",") if d]
    objs = []
    for src in B.SOURCES:
        obj = out / f"{name}_{src}.o"
        subprocess.run([B._nvcc(), *B.NVCC_FLAGS, *defs, "-c", str(B.CSRC / src), "-o", str(obj)], check=True)
        objs.append(str(obj))
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(out / f"{name}.so"), *objs, "-lpthread"], check=True)
    print(out / f"{name}.so")
