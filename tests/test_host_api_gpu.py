"""GPU tests of the host-side API surfaces above the kernels.

  * the C++ acceptance binary (tests/cpp/acceptance_cuda.cpp), which drives
    include/oilpaint_b200.hpp exactly like the reference's acceptance suite
    drives apply_sequential / apply_parallel;
  * the multi-device host path (opc_filter_rgb8_multi) with repeated device
    ordinals on one GPU: row bands and frame splits reassemble byte for byte;
  * the e2e pipelined host-pointer path on a large image (chunked H2D/D2H).
"""
from __future__ import annotations

import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle_lib
import paper_1405_1020_b200 as opc

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_cpp_acceptance_binary(gpu):
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], check=True)
    res = subprocess.run([str(ROOT / "build" / "acceptance_cuda"),
                          str(ROOT / "tests" / "golden" / "gradient8_r2_l20_zero.ppm")],
                         capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert res.stdout.count("PASS") == 4


@pytest.mark.parametrize("ndev", [2, 3, 8])
def test_multi_device_row_bands(gpu, ndev):
    rng = np.random.default_rng(ndev)
    img = rng.integers(0, 256, (413, 251, 3), dtype=np.uint8)
    for r, L, b in ((15, 20, 0), (5, 255, 1)):
        p = gpu.FilterParams(r, L, gpu.BorderPolicy(b))
        one = gpu.apply_cuda(img, p)
        many = gpu.apply_cuda(img, p, gpu.CudaConfig(devices=(0,) * ndev))
        assert np.array_equal(one, many)
        assert np.array_equal(one, oracle_lib.oracle_filter(img, r, L, b, threads=8))


def test_multi_device_frames(gpu):
    rng = np.random.default_rng(5)
    frames = rng.integers(0, 256, (7, 63, 95, 3), dtype=np.uint8)
    p = gpu.FilterParams(7, 30)
    a = gpu.apply_cuda_batch(frames, p)
    b = gpu.apply_cuda_batch(frames, p, gpu.CudaConfig(devices=(0, 0, 0)))
    assert np.array_equal(a, b)


def test_pipelined_host_path_large_image(gpu):
    """A > 48 MB image takes the chunked H2D / kernel / D2H pipeline."""
    img = gpu.generate(gpu.Pattern.NOISE, 6000, 3000, seed=11)
    p = gpu.FilterParams(15, 20)
    out = gpu.apply_cuda(img, p)
    # rows straddling chunk boundaries, checked against the oracle
    for y0 in (0, 180, 361, 1480, 2700, 3000 - 80):
        lo, hi = max(0, y0 - 15), min(3000, y0 + 80 + 15)
        sub = img[lo:hi, 2000:2400]
        want = oracle_lib.oracle_filter(np.ascontiguousarray(sub), 15, 20, 0, threads=8)
        got = out[lo:hi, 2000:2400]
        rows = slice(15 if lo > 0 else 0, (hi - lo) - (15 if hi < 3000 else 0))
        assert np.array_equal(got[rows, 15:-15], want[rows, 15:-15]), y0


@pytest.mark.gpu
@pytest.mark.parametrize("kind,seed", [(opc.Pattern.NOISE, 4), (opc.Pattern.NOISE, 42),
                                       (opc.Pattern.GRADIENT, 0), (opc.Pattern.UNIFORM, 0x123456),
                                       (opc.Pattern.CHECKER, 5), (opc.Pattern.SMOOTH, 2),
                                       (opc.Pattern.RECTS, 3), (opc.Pattern.VIDEO, 5)])
@pytest.mark.parametrize("w,h,offset", [(1, 1, 0), (333, 97, 0), (257, 3, 5), (1024, 64, 3)])
def test_generate_device_matches_host(gpu, kind, seed, w, h, offset):
    """On-device generation writes the host generator's bytes,
    also at unaligned destinations (VIDEO: frame 3 of the batch)."""
    import torch
    frame = 3 if kind == opc.Pattern.VIDEO else 0
    buf = torch.full((w * h * 3 + offset + 8,), 0xAB, dtype=torch.uint8, device="cuda")
    opc.generate_device(kind, w, h, buf.data_ptr() + offset, seed=seed, device=0,
                        stream=torch.cuda.current_stream().cuda_stream or None, frame=frame)
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    want = opc.generate(kind, w, h, seed=seed, frame=frame).reshape(-1)
    assert np.array_equal(got[offset:offset + want.size], want)
    assert (got[:offset] == 0xAB).all() and (got[offset + want.size:] == 0xAB).all()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_generate_device_full_config_inputs(gpu, name):
    """Full-size config inputs generated on the device hash to the committed
    input digests (tests/golden/config_digests.json)."""
    import hashlib
    import json
    import torch
    cfg = opc.CONFIGS[name]
    d = json.loads((Path(__file__).resolve().parent / "golden" / "config_digests.json").read_text())
    frames = [0, cfg.frames - 1] if cfg.frames > 1 else [0]
    buf = torch.empty(cfg.width * cfg.height * 3, dtype=torch.uint8, device="cuda")
    for f in frames:
        opc.generate_device(cfg.pattern, cfg.width, cfg.height, buf.data_ptr(), seed=cfg.seed,
                            device=0, frame=f)
        torch.cuda.synchronize()
        assert hashlib.sha256(buf.cpu().numpy().tobytes()).hexdigest() == d[name]["inputs"][f], (name, f)


def test_kernel_timing_records_each_launch(gpu):
    """opc_kernel_timing: CUDA events around every kernel launch (bench.py's
    roofline uses the dominant kernel's measured time)."""
    from paper_1405_1020_b200 import _lib
    img = opc.generate(opc.Pattern.NOISE, 700, 300, seed=5)
    p = opc.FilterParams(7, 20)
    skew = opc.CudaConfig(kernel=_lib.OPC_KERNEL_SKEW)
    opc.kernel_timing(True)
    for _ in range(3):
        opc.apply_cuda(img, p, skew)
    opc.apply_cuda(img, p)  # automatic choice for this size: the bit-plane family
    opc.apply_cuda(img, p, opc.CudaConfig(kernel=_lib.OPC_KERNEL_COLUMN))
    skew_ms, skew_n = opc.kernel_timing_read(_lib.OPC_KID_SKEW)
    pre_ms, pre_n = opc.kernel_timing_read(_lib.OPC_KID_PREPASS)
    bor_ms, bor_n = opc.kernel_timing_read(_lib.OPC_KID_BORDER)
    col_ms, col_n = opc.kernel_timing_read(_lib.OPC_KID_COLUMN)
    pl_ms, pl_n = opc.kernel_timing_read(_lib.OPC_KID_PLANES)
    opc.kernel_timing(False)
    # the border job rides on the shear pre-pass / the column and bit-plane
    # kernels: no border launch of its own
    assert (skew_n, pre_n, bor_n, col_n, pl_n) == (3, 3, 0, 1, 1)
    assert skew_ms > 0 and pre_ms > 0 and bor_ms == 0 and col_ms > 0 and pl_ms > 0
    opc.apply_cuda(img, p, skew)  # timing off: nothing recorded
    assert opc.kernel_timing_read(_lib.OPC_KID_SKEW) == (0.0, 0)


@pytest.mark.parametrize("y0,y1", [(0, 40), (37, 151), (150, 203), (0, 203)])
def test_band_writes_exactly_its_rows(gpu, y0, y1):
    """Canary (proj/tests/test_parallel.cpp:65-103 lifted to the band call): the
    band's output rows are all written -- identical results over 0x00- and
    0xFF-filled buffers -- nothing outside them is, and the rows equal the
    whole-image result."""
    import ctypes
    from paper_1405_1020_b200._lib import LIB
    img = opc.generate(opc.Pattern.NOISE, 97, 203, seed=8)
    p = opc.FilterParams(6, 20)
    whole = opc.apply_cuda(img, p)
    lo, hi = opc.band_input_rows(203, y0, y1, 6)
    src = np.ascontiguousarray(img[lo:hi])
    outs = []
    for fill in (0x00, 0xFF):
        buf = np.full((y1 - y0 + 2) * 97 * 3, fill, np.uint8)  # one guard row each side
        c = opc.CudaConfig().to_c()
        rc = LIB.opc_filter_rgb8_band(src.ctypes.data, buf.ctypes.data + 97 * 3, 97, 203, y0, y1,
                                      6, 20, 0, ctypes.byref(c))
        assert rc == 0, LIB.opc_last_error()
        assert (buf[:97 * 3] == fill).all() and (buf[-97 * 3:] == fill).all()
        outs.append(buf[97 * 3:-97 * 3].reshape(y1 - y0, 97, 3))
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], whole[y0:y1])


@pytest.mark.parametrize("kernel", ["skew", "slide"])
def test_two_streams_share_scratch_safely(gpu, kernel):
    """Device-pointer calls in flight on two user streams at once (and a host
    call on the library's own stream) share the device's scratch plane: each
    launch is ordered after the previous scratch user, so no call reads the
    other's sheared / transposed plane (capi.cu scratch events)."""
    import torch
    from paper_1405_1020_b200 import _lib
    L = 20 if kernel == "skew" else 100
    kid = _lib.OPC_KERNEL_SKEW if kernel == "skew" else _lib.OPC_KERNEL_SLIDE
    imgs = [gpu.generate(gpu.Pattern.NOISE, 1500, 700, seed=s) for s in (1, 2, 3, 4)]
    p = gpu.FilterParams(9, L)
    want = [gpu.apply_cuda(im, p, gpu.CudaConfig(kernel=kid)) for im in imgs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    d_in = [torch.from_numpy(im).cuda() for im in imgs]
    torch.cuda.synchronize()
    d_out = [torch.empty_like(t) for t in d_in]
    for rep in range(3):
        for i in range(4):
            s = streams[i % 2]
            cfg = gpu.CudaConfig(device=0, stream=s.cuda_stream, kernel=kid)
            gpu.apply_cuda_device(d_in[i].data_ptr(), d_out[i].data_ptr(), 1500, 700, p, cfg)
        host = gpu.apply_cuda(imgs[rep], p, gpu.CudaConfig(kernel=kid))  # ctx stream, blocking
        assert np.array_equal(host, want[rep])
        torch.cuda.synchronize()
        for i in range(4):
            assert np.array_equal(d_out[i].cpu().numpy(), want[i]), (rep, i)


def test_small_frame_batch_units(gpu):
    """A long batch of small frames runs in bounded units (about 48 MB of frames
    each, pinned staging sized to one unit) and equals the per-frame results
    and the oracle, from pageable and from pinned buffers."""
    import torch
    frames = gpu.generate(gpu.Pattern.NOISE, 640, 480, seed=21)
    batch = np.stack([np.roll(frames, 7 * k, axis=1) for k in range(60)])  # 55 MB > one unit
    p = gpu.FilterParams(2, 20)
    got = gpu.apply_cuda_batch(batch, p)
    for k in (0, 1, 51, 52, 59):
        assert np.array_equal(got[k], gpu.apply_cuda(batch[k], p)), k
    assert np.array_equal(got[59], oracle_lib.oracle_filter(batch[59], 2, 20, 0))
    pinned = torch.from_numpy(batch).pin_memory().numpy()
    assert np.array_equal(gpu.apply_cuda_batch(pinned, p), got)


def test_multi_device_frames_match_oracle(gpu):
    rng = np.random.default_rng(9)
    frames = rng.integers(0, 256, (5, 41, 77, 3), dtype=np.uint8)
    got = gpu.apply_cuda_batch(frames, gpu.FilterParams(7, 30), gpu.CudaConfig(devices=(0, 0)))
    for k in range(5):
        assert np.array_equal(got[k], oracle_lib.oracle_filter(frames[k], 7, 30, 0)), k


def test_c4_input_is_reference_noise(gpu):
    """The C4 bench input (Noise{4}, 16384 wide) equals the reference generator
    (proj/src/pattern.cpp:64-76 via oracle/_ref) on a band of rows."""
    if not oracle_lib.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = oracle_lib.load_ref()
    want = np.empty((64, 16384, 3), np.uint8)
    assert ref.ref_generate(0, 4, 16384, 64, want.ctypes.data) == 0
    got = gpu.generate(gpu.Pattern.NOISE, 16384, 64, seed=4)
    assert np.array_equal(got, want)
