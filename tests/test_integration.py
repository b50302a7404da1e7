"""The B200 engine inside the reference's own code.

integration/ compiles oilpaint::apply_cuda (integration/include/oilpaint/cuda.hpp,
integration/src/cuda.cpp) against the REFERENCE headers -- the reference's
oilpaint::Image, FilterParams and validate -- and builds two reference
programs from the staged reference sources with integration/patches/
engine-cuda.patch applied (integration/Makefile):

  ref_acceptance_cuda  proj/tests/acceptance.cpp with apply_cuda checked beside
                       apply_sequential / apply_parallel in criteria 1, 2, 6
                       (acceptance.cpp:44-67, 71-101, 196-218)
  sweep_cuda           run_sweep / write_csv (proj/src/bench.cpp:78-166) with
                       EngineKind::Cuda (bench.hpp:12) as the contender

CPU tests: the programs are built, link the product library, and reject bad
arguments the reference way; the patch still applies to the reference.  GPU
tests run them.
"""
from __future__ import annotations

import csv
import io
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "build" / "integration"
ACCEPT = OUT / "ref_acceptance_cuda"
SWEEP = OUT / "sweep_cuda"
REF = Path("/root/reference/proj")


@pytest.fixture(scope="module")
def built():
    if REF.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "integration")], check=True)
    if not (ACCEPT.exists() and SWEEP.exists()):
        pytest.fail("build/integration binaries missing: run __graft_entry__.build() where "
                    "/root/reference is present")
    return True


def test_programs_link_the_product_library(built):
    for exe in (ACCEPT, SWEEP):
        ldd = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
        assert "liboilpaint_b200.so" in ldd and "not found" not in ldd, ldd
        syms = subprocess.run(["nm", "-C", str(exe)], capture_output=True, text=True).stdout
        # the reference's own engines and the adapter, in one program
        assert "oilpaint::apply_cuda(oilpaint::Image const&" in syms
        assert "oilpaint::apply_sequential(oilpaint::Image const&" in syms
        assert "oilpaint::validate(oilpaint::Image const&" in syms


@pytest.mark.skipif(not REF.exists(), reason="needs /root/reference")
def test_patch_applies_to_the_reference(tmp_path):
    for sub in ("include", "src", "tests"):
        (tmp_path / sub).mkdir()
    subprocess.run(["cp", "-r", str(REF / "include/oilpaint"), str(tmp_path / "include")], check=True)
    subprocess.run(["cp", str(REF / "src/bench.cpp"), str(tmp_path / "src")], check=True)
    subprocess.run(["cp", str(REF / "tests/acceptance.cpp"), str(tmp_path / "tests")], check=True)
    subprocess.run(["chmod", "-R", "u+w", str(tmp_path)], check=True)
    res = subprocess.run(["patch", "-p1", "--dry-run", "-d", str(tmp_path)],
                         stdin=open(ROOT / "integration/patches/engine-cuda.patch"),
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAILED" not in res.stdout and "fuzz" not in res.stdout


def test_sweep_rejects_bad_arguments(built):
    for args, rc in ((["--sizes", "huge"], 3), (["--engine", "gpu"], 3), (["--reps"], 3)):
        res = subprocess.run([str(SWEEP), *args], capture_output=True, text=True, timeout=60)
        assert res.returncode == rc, (args, res.stderr)


@pytest.mark.gpu
def test_reference_acceptance_with_apply_cuda(built, gpu):
    """The reference acceptance suite, its criteria 1, 2 and 6 extended with
    oilpaint::apply_cuda on oilpaint::Image: all criteria PASS."""
    res = subprocess.run([str(ACCEPT)], capture_output=True, text=True, timeout=900)
    print(res.stdout)
    lines = {int(ln.split()[2]): ln for ln in res.stdout.splitlines()
             if ln[:4] in ("PASS", "FAIL", "SKIP") and "criterion" in ln}
    for k in (1, 2, 6):
        assert lines[k].startswith("PASS"), lines[k]
    assert "(seq and cuda)" in lines[1]
    assert "cuda bands {1,2,4,8}" in lines[2]
    assert "all three engines" in lines[6]
    assert res.returncode == 0, res.stdout + res.stderr


@pytest.mark.gpu
def test_reference_sweep_with_engine_cuda(built, gpu):
    """run_sweep with EngineKind::Cuda: the reference CSV with 'cuda' rows and
    the seq-vs-cuda improvement_pct pairs (the paper's table with a GPU column)."""
    res = subprocess.run([str(SWEEP), "--sizes", "vga,xga", "--radii", "2,8", "--reps", "3"],
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr
    records, pairs = res.stdout.split("\n\n")
    rows = list(csv.DictReader(io.StringIO(records)))
    assert [(r["label"], r["radius"], r["engine"]) for r in rows] == [
        ("VGA", "2", "seq"), ("VGA", "2", "cuda"), ("VGA", "8", "seq"), ("VGA", "8", "cuda"),
        ("XGA", "2", "seq"), ("XGA", "2", "cuda"), ("XGA", "8", "seq"), ("XGA", "8", "cuda")]
    prs = list(csv.DictReader(io.StringIO(pairs)))
    assert len(prs) == 4
    for p in prs:
        t1, t2, pct = float(p["t1_ms"]), float(p["t2_ms"]), float(p["improvement_pct"])
        assert abs(pct - 100 * (t1 - t2) / t1) < 1e-4
        assert pct > 90, p  # the GPU engine is far faster than one CPU core
