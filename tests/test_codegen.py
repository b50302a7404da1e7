"""Build-level guards on the hot kernels' code generation (CPU: cuobjdump on
the in-tree library).  Round 2 found the C4 skew kernel 14% slower after an
unrelated change to a shared header altered its register allocation; the
timing tests catch a slowdown only on the GPU box, these catch the usual
cause here: spills to local memory on the kernels the five configs run."""
from __future__ import annotations

import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1405_1020_b200" / "liboilpaint_b200.so"

# mangled-name fragment -> (what runs it, register ceiling, stack ceiling)
# (the 31-bin skew kernel has carried 32 bytes of stack since round 1: its
# 16-bin window path at the 168-register launch bound, profiles/r01_notes.md)
HOT = {
    "skew_kernelILi21ELi96ELb0E": ("C4 (r=15, 21 bins)", 168, 0),
    "skew_kernelILi31ELi64ELb1E": ("C5 (r=7, 31 bins, KEY layout)", 168, 32),
    "planes_kernelILi5ELb1ELb0E": ("C2 (r=5, TMA tile, per-warp sums)", 168, 0),
    "planes_kernelILi2ELb1ELb0E": ("C1 (r=2, TMA tile, per-warp sums)", 168, 0),
    "planes_kernelILi7ELb1ELb1E": ("r=7 multi-round launches", 168, 0),
    "shear_kernelILb1E": ("C4 / C5 pre-pass (TMA tiles)", 64, 0),
}


def resource_usage() -> dict[str, tuple[int, int]]:
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", str(LIB)], capture_output=True,
                         text=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and name:
            res[name] = (int(m.group(1)), int(m.group(2)))
            name = None
    return res


@pytest.mark.skipif(shutil.which("cuobjdump") is None or not LIB.exists(),
                    reason="needs cuobjdump and the built library")
def test_hot_kernels_do_not_spill():
    res = resource_usage()
    for frag, (what, reg_max, stack_max) in HOT.items():
        hits = [(n, v) for n, v in res.items() if frag in n]
        assert hits, f"{frag} ({what}) not in the library"
        for n, (reg, stack) in hits:
            assert stack <= stack_max, f"{what}: {n} spills ({stack} bytes of stack)"
            assert reg <= reg_max, f"{what}: {n} uses {reg} registers"
