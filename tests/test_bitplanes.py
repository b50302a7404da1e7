"""Host check of the bit-plane kernel family's counter arithmetic
(paper_1405_1020_b200/csrc/bitplanes.cuh): compiles tests/cpp/bitplanes_test.cpp
with g++ and runs it -- carry-save row histograms, the fused window update and
the plane-walk argmax against plain per-bin integers (the reference's
lowest-index strict-> argmax, filter.hpp:71-82).  The CUDA kernels built on
them are checked on the GPU by tests/test_parity_gpu.py."""
from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_bitplane_counters_match_integer_histograms(tmp_path):
    exe = tmp_path / "bitplanes_test"
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wno-unknown-pragmas", "-I",
                    str(ROOT / "paper_1405_1020_b200" / "csrc"),
                    str(ROOT / "tests" / "cpp" / "bitplanes_test.cpp"), "-o", str(exe)], check=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failures" in res.stdout
