"""In-tree build of the product library paper_1405_1020_b200/liboilpaint_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo (sm_100a only, no other
targets), one object per source compiled in parallel, linked with the static
CUDA runtime.  The .so is git-ignored but travels to the GPU box with the
gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "obj"
LIB = PKG / "liboilpaint_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr", "-I", str(ROOT / "include")] + ARCH
SOURCES = ["capi.cu", "direct.cu", "column.cu", "planes.cu", "skew.cu", "slide.cu", "gen.cu", "patterns.cpp"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build liboilpaint_b200.so")


def _compile(src: Path, obj: Path, verbose: bool) -> None:
    cmd = [_nvcc(), *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    # every header a source can include: csrc/*.cuh, csrc/*.h (gen_spec.h is
    # shared by gen.cu and patterns.cpp) and the public include/*.h
    headers = (list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) +
               list((ROOT / "include").glob("*.h")))
    jobs = []
    objs = []
    for name in SOURCES:
        src = CSRC / name
        obj = BUILD / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *headers]):
            jobs.append((src, obj))
    with cf.ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        list(ex.map(lambda j: _compile(j[0], j[1], verbose), jobs))
    if force or jobs or _stale(LIB, objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


def build_variant(out: Path, defines: list[str]) -> Path:
    """An experiment build of the library with extra -D flags (A/B runs and
    instrumented builds; load it with OILPAINT_B200_LIB=<out>).  Objects go
    to build/var_<name>/."""
    out = Path(out)
    objdir = ROOT / "build" / ("var_" + out.stem)
    objdir.mkdir(parents=True, exist_ok=True)
    flags = [f"-D{d}" for d in defines]
    def one(name):
        obj = objdir / (name + ".o")
        cmd = [_nvcc(), *NVCC_FLAGS, *flags, "-c", str(CSRC / name), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {name}:\n{res.stdout}\n{res.stderr}")
        return obj
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(one, SOURCES))
    cmd = [_nvcc(), *ARCH, "-shared", "-o", str(out), *map(str, objs), "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return out


TOOL_SRC = ROOT / "tools" / "oilbench_cuda.cpp"
TOOL = ROOT / "build" / "oilbench_cuda"


def build_tools(force: bool = False) -> Path:
    """The CLI front end (tools/oilbench_cuda.cpp), host C++ over the C-ABI,
    linked against the in-tree library (rpath $ORIGIN/../paper_1405_1020_b200)."""
    lib = build(force)
    deps = [TOOL_SRC, lib, *(ROOT / "include").glob("*.h*")]
    if force or _stale(TOOL, deps):
        TOOL.parent.mkdir(parents=True, exist_ok=True)
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-std=c++20", "-O2", "-Wall", "-I", str(ROOT / "include"), str(TOOL_SRC),
               "-o", str(TOOL), "-L", str(PKG), "-loilpaint_b200",
               "-Wl,-rpath,$ORIGIN/../paper_1405_1020_b200"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"building {TOOL.name} failed:\n{res.stdout}\n{res.stderr}")
    return TOOL


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_tools()
    print(LIB)
    print(TOOL)
