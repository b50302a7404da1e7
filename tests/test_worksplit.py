"""Host check of the persistent kernels' work split (csrc/worksplit.cuh).

Compiles tests/cpp/worksplit_test.cpp with g++ and runs it: for ~3000 launch
shapes (frames, bands, interior width, blocks, warps per block, static share)
every (frame, band, column) unit is covered by exactly one pass, and no pass
crosses a band end.  (The kernels' results at real sizes are checked on the GPU
by tests/test_parity_gpu.py and tests/test_configs_gpu.py.)
"""
from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_worksplit_covers_every_unit_once(tmp_path):
    exe = tmp_path / "worksplit_test"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", str(ROOT / "paper_1405_1020_b200" / "csrc"),
                    str(ROOT / "tests" / "cpp" / "worksplit_test.cpp"), "-o", str(exe)], check=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failures" in res.stdout
