"""The CLI front end tools/oilbench_cuda.cpp.

Mirrors the reference CLI contract (proj/tools/oilbench.cpp): subcommands
apply / gen / bench over binary PPM files and exit codes 0 ok, 1 usage, 2 I/O,
parse or runtime error, 3 filter parameter error.  The PPM codec
(include/oilpaint_b200_ppm.hpp) keeps the reference's byte format
(proj/include/oilpaint/ppm.hpp); its error messages name the offending part
(magic, width, height, maxval, payload), the substrings the reference tests pin
(proj/tests/test_ppm.cpp:44-59).  CPU tests cover
argument handling, generation and PPM parsing (a well-formed file reaches the
engine, which then reports that no CUDA device is present); the GPU tests run
the filter and the sweep.
"""
from __future__ import annotations

import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle_lib
import paper_1405_1020_b200 as opc
from paper_1405_1020_b200 import build as B

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def tool() -> Path:
    return B.build_tools()


def run(tool, *args, check_rc=None):
    res = subprocess.run([str(tool), *map(str, args)], capture_output=True, text=True, timeout=600)
    if check_rc is not None:
        assert res.returncode == check_rc, (res.returncode, res.stdout, res.stderr)
    return res


def read_ppm(path: Path) -> np.ndarray:
    data = path.read_bytes()
    head, rest = data.split(b"\n", 1)
    assert head == b"P6"
    dims, rest = rest.split(b"\n", 1)
    w, h = map(int, dims.split())
    maxval, payload = rest.split(b"\n", 1)
    assert maxval == b"255"
    return np.frombuffer(payload, np.uint8).reshape(h, w, 3)


def write_ppm(path: Path, img: np.ndarray) -> None:
    h, w, _ = img.shape
    path.write_bytes(b"P6\n%d %d\n255\n" % (w, h) + img.tobytes())


def test_usage_errors_exit_1(tool):
    for args in ([], ["frobnicate"], ["apply"], ["apply", "--input", "x.ppm"],
                 ["apply", "--input", "a", "--output", "b", "--bogus", "1"],
                 ["apply", "--input", "a", "--output", "b", "--levels", "0"],
                 ["apply", "--input", "a", "--output", "b", "--levels", "256"],
                 ["apply", "--input", "a", "--output", "b", "--radius", "-1"],
                 ["apply", "--input", "a", "--output", "b", "--engine", "seq"],
                 ["apply", "--input", "a", "--output", "b", "--border", "mirror"],
                 ["gen", "--pattern", "plaid", "--width", "4", "--height", "4", "--output", "x"],
                 ["gen", "--pattern", "noise", "--width", "0", "--height", "4", "--output", "x"],
                 ["bench", "--sizes", "huge"], ["bench", "--reps", "0"],
                 ["apply", "--input", "a", "--output", "b", "--threads", "4"],
                 ["bench", "--threads=8"]):
        res = run(tool, *args)
        assert res.returncode == 1, (args, res.stderr)
        assert "usage:" in res.stderr
    assert run(tool, "--help").returncode == 0


def test_gen_patterns(tool, tmp_path):
    p = tmp_path / "n.ppm"
    run(tool, "gen", "--pattern", "noise", "--width", 4, "--height", 1, "--seed", 42,
        "--output", p, check_rc=0)
    # reference Noise{42} byte stream, pinned by proj/tests/test_pattern.cpp:43-50
    assert read_ppm(p).reshape(-1).tolist() == [0x95, 0x6E, 0xEB, 0x2F, 0x26, 0x32, 0xD7, 0xBD,
                                                0x03, 0xF1, 0x66, 0xB2]
    run(tool, "gen", "--pattern", "noise", "--width", 33, "--height", 17, "--seed", 7,
        "--output", p, check_rc=0)
    assert np.array_equal(read_ppm(p), opc.generate(opc.Pattern.NOISE, 33, 17, seed=7))
    run(tool, "gen", "--pattern", "uniform", "--width", 5, "--height", 3, "--output", p, check_rc=0)
    assert (read_ppm(p) == 128).all()
    run(tool, "gen", "--pattern", "checker", "--width", 20, "--height", 10, "--output", p,
        check_rc=0)
    img = read_ppm(p)
    yy, xx = np.mgrid[0:10, 0:20]
    want = np.where(((xx // 8 + yy // 8) % 2 == 0), 255, 0).astype(np.uint8)
    assert np.array_equal(img, np.repeat(want[:, :, None], 3, axis=2))
    run(tool, "gen", "--pattern", "gradient", "--width", 13, "--height", 5, "--output", p,
        check_rc=0)
    g = np.empty((5, 13, 3), np.uint8)
    oracle_lib.oracle().oracle_gradient(13, 5, g.ctypes.data)
    assert np.array_equal(read_ppm(p), g)
    assert p.read_bytes().startswith(b"P6\n13 5\n255\n")  # canonical header (ppm.hpp write_ppm)


def _engine_reached(res) -> bool:
    """The input parsed and validated: the engine ran (GPU) or reported no device."""
    return res.returncode == 0 or "no CUDA device" in res.stderr


@pytest.mark.parametrize("blob,ok,msg", [
    (b"P6\n8 8\n255\n" + bytes(192), True, ""),
    (b"P6 8 8 255 " + bytes(192), True, ""),
    (b"P6\n# comment\n8 # w\n8\n255\n" + bytes(192) + b"trailing", True, ""),
    (b"P3\n8 8\n255\n" + bytes(192), False, "magic"),
    (b"P6x8 8\n255\n" + bytes(192), False, "magic"),
    (b"P6\n8 8\n65535\n" + bytes(384), False, "maxval"),
    (b"P6\n8 8\n255\n" + bytes(100), False, "payload too short"),
    (b"P6\n0 8\n255\n", False, "width must be at least 1"),
    (b"P6\n8 0\n255\n", False, "height must be at least 1"),
    (b"P6\n8 x\n255\n", False, "height is not a decimal number"),
    (b"P6\n99999999999 8\n255\n", False, "width is too large"),
    (b"P6\n8 8", False, "header ends before the maxval"),
    (b"P6\n8 8\n255", False, "maxval must be followed by one whitespace byte"),
])
def test_ppm_parsing(tool, tmp_path, blob, ok, msg):
    src = tmp_path / "in.ppm"
    src.write_bytes(blob)
    res = run(tool, "apply", "--input", src, "--output", tmp_path / "o.ppm", "--radius", 1)
    if ok:
        assert _engine_reached(res), res.stderr
    else:
        assert res.returncode == 2 and msg in res.stderr, (res.returncode, res.stderr)


def test_parameter_errors_exit_3(tool, tmp_path):
    src = tmp_path / "in.ppm"
    write_ppm(src, np.zeros((8, 8, 3), np.uint8))
    res = run(tool, "apply", "--input", src, "--output", tmp_path / "o.ppm", "--radius", 4)
    assert res.returncode == 3 and "leaves no interior" in res.stderr


def test_missing_input_exit_2(tool, tmp_path):
    res = run(tool, "apply", "--input", tmp_path / "nope.ppm", "--output", tmp_path / "o.ppm")
    assert res.returncode == 2 and "cannot open" in res.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("border", ["copy", "zero"])
def test_apply_matches_oracle(tool, tmp_path, border, gpu):
    img = opc.generate(opc.Pattern.NOISE, 67, 45, seed=3)
    src, dst = tmp_path / "in.ppm", tmp_path / "out.ppm"
    write_ppm(src, img)
    res = run(tool, "apply", "--input", src, "--output", dst, "--radius", 3, "--levels", 12,
              "--border", border, check_rc=0)
    assert "time_process_ms=" in res.stderr
    want = oracle_lib.oracle_filter(img, 3, 12, 0 if border == "copy" else 1)
    assert np.array_equal(read_ppm(dst), want)


@pytest.mark.gpu
def test_bench_sweep_csv(tool, tmp_path, gpu):
    base = tmp_path / "ref.csv"
    base.write_text("label,width,height,radius,levels,engine,reps,median_ms,min_ms,max_ms\n"
                    "VGA,640,480,2,20,seq,5,54.000000,53.000000,55.000000\n"
                    "VGA,640,480,2,20,par,5,7.500000,7.000000,8.000000\n"
                    "\nlabel,radius,t1_ms,t2_ms,improvement_pct\n"
                    "VGA,2,54.000000,7.500000,86.111111\n")
    out = tmp_path / "cuda.csv"
    run(tool, "bench", "--sizes", "vga,96x64", "--radii", "2,3", "--reps", 3, "--out", out,
        "--baseline", base, check_rc=0)
    records, pairs = out.read_text().split("\n\n")
    rows = [r.split(",") for r in records.strip().split("\n")[1:]]
    assert [(r[0], r[3], r[5], r[6]) for r in rows] == [
        ("VGA", "2", "cuda", "3"), ("VGA", "3", "cuda", "3"),
        ("96x64", "2", "cuda", "3"), ("96x64", "3", "cuda", "3")]
    for r in rows:
        med, lo, hi = map(float, r[7:10])
        assert 0 < lo <= med <= hi
    prow = pairs.strip().split("\n")
    assert prow[0] == "label,radius,t1_ms,t2_ms,improvement_pct" and len(prow) == 2
    label, radius, t1, t2, imp = prow[1].split(",")
    assert (label, radius, float(t1)) == ("VGA", "2", 54.0)
    assert abs(float(imp) - 100 * (54.0 - float(t2)) / 54.0) < 1e-3


def test_ppm_bytes_match_reference_writer(tool, tmp_path):
    """The codec's canonical bytes equal the reference write_ppm (proj/src/ppm.cpp
    via oracle/_ref) for generated images of several shapes."""
    if not oracle_lib.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = oracle_lib.load_ref()
    for w, h, seed in ((1, 1, 0), (33, 17, 7), (640, 3, 9)):
        p = tmp_path / "g.ppm"
        run(tool, "gen", "--pattern", "noise", "--width", w, "--height", h, "--seed", seed,
            "--output", p, check_rc=0)
        img = np.empty((h, w, 3), np.uint8)
        assert ref.ref_generate(0, seed, w, h, img.ctypes.data) == 0
        buf = np.empty(64 + img.size, np.uint8)
        n = ref.ref_write_ppm(img.ctypes.data, w, h, buf.ctypes.data, buf.size)
        assert p.read_bytes() == buf[:n].tobytes()
