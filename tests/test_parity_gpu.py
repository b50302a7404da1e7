"""GPU parity suite: the CUDA product path through the C-ABI vs the oracle.

Mirrors the reference's own tests:
  * acceptance criterion 1 (proj/tests/acceptance.cpp:44-67) -- 1000 random
    small cases vs the brute-force oracle, bit exact;
  * criterion 2 (acceptance.cpp:71-101) -- 200 cases up to 128x128, r <= 5;
  * criterion 6 / test_filter.cpp:205-211 -- the golden 8x8 gradient PPM;
  * test_filter.cpp known answers, invariants, border policy, validation;
  * test_parallel.cpp's partition checks, with GPU row bands in place of worker
    chunks (every output row produced exactly once, bands == whole image).
Every kernel family is also forced on every case it accepts.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import oracle_lib
from test_oracle import load_cases, ppm_payload

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
AUTO, DIRECT, SKEW, SLIDE, COLUMN, PLANES = 0, 1, 2, 3, 4, 5


def run(opc, img, r, L, border=0, kernel=AUTO, allow256=False):
    cfg = opc.CudaConfig(kernel=kernel, allow_levels_256=allow256)
    return opc.apply_cuda(img, opc.FilterParams(r, L, opc.BorderPolicy(border)), cfg)


def skew_ok(r, L):
    return L + 1 <= 32 and r <= 15


def slide_ok(r, L):
    return r <= 15


def column_ok(r, L):
    return L + 1 <= 32 and r <= 7


def planes_ok(r, L):
    return L + 1 <= 32 and 1 <= r <= 7


def test_reference_fixture_cases_all_kernels(gpu):
    n = 0
    for w, h, r, L, border, src, img, want in load_cases():
        allow = L == 256
        assert np.array_equal(run(gpu, img, r, L, border, AUTO, allow), want), (w, h, r, L, border)
        assert np.array_equal(run(gpu, img, r, L, border, DIRECT, allow), want), (w, h, r, L)
        if skew_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, border, SKEW), want), (w, h, r, L, border)
        if slide_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, border, SLIDE, allow), want), (w, h, r, L)
        if column_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, border, COLUMN), want), (w, h, r, L, border)
        if planes_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, border, PLANES), want), (w, h, r, L, border)
        n += 1
    assert n == 296


def test_golden_ppm(gpu):
    _, _, golden = ppm_payload(GOLDEN / "gradient8_r2_l20_zero.ppm")
    img = gpu.generate(gpu.Pattern.GRADIENT, 8, 8)
    for k in (AUTO, DIRECT, SKEW, SLIDE, COLUMN, PLANES):
        assert np.array_equal(run(gpu, img, 2, 20, 1, k), golden)


def test_criterion1_random_small_vs_oracle(gpu):
    rng = np.random.default_rng(101)
    for i in range(1000):
        w, h = int(rng.integers(1, 17)), int(rng.integers(1, 17))
        r = int(rng.integers(0, min(3, (min(w, h) - 1) // 2) + 1))
        L = int(rng.choice([1, 10, 20, 255]))
        b = int(rng.integers(0, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        want = oracle_lib.oracle_filter(img, r, L, b)
        assert np.array_equal(run(gpu, img, r, L, b), want), (i, w, h, r, L, b)


def test_criterion2_random_medium_vs_oracle(gpu):
    rng = np.random.default_rng(202)
    for i in range(200):
        w, h = int(rng.integers(1, 129)), int(rng.integers(1, 129))
        r = int(rng.integers(0, min(5, (min(w, h) - 1) // 2) + 1))
        L = int(rng.choice([1, 20, 30, 255]))
        b = int(rng.integers(0, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        want = oracle_lib.oracle_filter(img, r, L, b, threads=4)
        assert np.array_equal(run(gpu, img, r, L, b), want), (i, w, h, r, L, b)
        if skew_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, b, SKEW), want), (i, w, h, r, L, b)
        if column_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, b, COLUMN), want), (i, w, h, r, L, b)
        if planes_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, b, PLANES), want), (i, w, h, r, L, b)


@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("L", [1, 2, 15, 20, 23, 30, 31])
def test_planes_radius_levels_grid(gpu, r, L):
    """Bit-plane family: every radius it instantiates (the row loop is
    unrolled by 2r+1), counts up to (2r+1)^2 in its bit planes, 2..32 bins,
    ragged widths (partial 128-column blocks and 32-column warps) and heights
    (partial row blocks)."""
    rng = np.random.default_rng(r * 1000 + L + 7)
    h = 2 * r + 1 + int(rng.integers(0, 300))
    w = 2 * r + 1 + int(rng.integers(0, 400))
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    for b in (0, 1):
        want = oracle_lib.oracle_filter(img, r, L, b, threads=4)
        assert np.array_equal(run(gpu, img, r, L, b, PLANES), want), (r, L, b, w, h)


@pytest.mark.parametrize("r", [0, 1, 2, 3, 5, 7])
@pytest.mark.parametrize("L", [1, 2, 15, 20, 23, 30, 31])
def test_column_radius_levels_grid(gpu, r, L):
    rng = np.random.default_rng(r * 10000 + L)
    h = 2 * r + 1 + int(rng.integers(0, 300))
    w = 2 * r + 1 + int(rng.integers(0, 400))
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    for b in (0, 1):
        want = oracle_lib.oracle_filter(img, r, L, b, threads=4)
        assert np.array_equal(run(gpu, img, r, L, b, COLUMN), want), (r, L, b, w, h)


@pytest.mark.parametrize("r", [0, 1, 2, 5, 7, 10, 14, 15])
@pytest.mark.parametrize("L", [1, 2, 7, 11, 20, 23, 30, 31])
def test_skew_radius_levels_grid(gpu, r, L):
    rng = np.random.default_rng(r * 100 + L)
    h = 2 * r + 1 + int(rng.integers(0, 70))
    w = 2 * r + 1 + int(rng.integers(0, 300))
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    want = oracle_lib.oracle_filter(img, r, L, 0, threads=4)
    assert np.array_equal(run(gpu, img, r, L, 0, SKEW), want)


@pytest.mark.parametrize("r", [0, 1, 3, 10, 15])
@pytest.mark.parametrize("L", [31, 40, 100, 255, 256])
def test_slide_radius_levels_grid(gpu, r, L):
    rng = np.random.default_rng(r * 1000 + L)
    h = 2 * r + 1 + int(rng.integers(0, 70))
    w = 2 * r + 1 + int(rng.integers(0, 300))
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    want = oracle_lib.oracle_filter(img, r, L, 0, threads=4)
    assert np.array_equal(run(gpu, img, r, L, 0, SLIDE, L == 256), want)
    if L + 1 > 32:
        assert np.array_equal(run(gpu, img, r, L, 0, AUTO, L == 256), want)


@pytest.mark.parametrize("L", [20, 255, 256])
def test_slide_rectangles_and_ties(gpu, L):
    """C3-like content: flat rectangles (winner changes at edges), plus
    two-tone noise with many exact ties and pure white (bin L)."""
    rng = np.random.default_rng(L)
    img = gpu.generate(gpu.Pattern.RECTS, 300, 180, seed=L)
    for r in (1, 4, 10, 15):
        want = oracle_lib.oracle_filter(img, r, L, 0, threads=4)
        assert np.array_equal(run(gpu, img, r, L, 0, SLIDE, L == 256), want), r
    two = np.where(rng.random((90, 170, 1)) < 0.5, 255, 0).astype(np.uint8).repeat(3, 2)
    for r in (2, 7):
        want = oracle_lib.oracle_filter(two, r, L, 1, threads=4)
        assert np.array_equal(run(gpu, two, r, L, 1, SLIDE, L == 256), want), r


@pytest.mark.parametrize("content", ["h_stripes", "v_stripes", "sparse_edges", "thin_stripes", "corners"])
def test_slide_structured_content(gpu, content):
    """The content-dependent paths of the slide family: striped pass starts
    (every column equal / every column one colour), long flat stretches jumped
    without ring loads, steps whose rows form one, two or many runs of a bin
    pair, winner changes of many lanes to one bin (shared row sums)."""
    rng = np.random.default_rng(len(content))
    h, w = 150, 1300
    img = np.empty((h, w, 3), np.uint8)
    img[:] = rng.integers(0, 256, 3, dtype=np.uint8)
    if content == "h_stripes":
        for y in range(0, h, 23):
            img[y:y + int(rng.integers(1, 12))] = rng.integers(0, 256, 3, dtype=np.uint8)
    elif content == "v_stripes":
        for x in range(0, w, 57):
            img[:, x:x + int(rng.integers(1, 30))] = rng.integers(0, 256, 3, dtype=np.uint8)
    elif content == "sparse_edges":  # a few edges, hundreds of flat columns between them
        for x in (5, 400, 401, 1000, 1290):
            img[:, x:] = rng.integers(0, 256, 3, dtype=np.uint8)
        img[70:, 600:900] = rng.integers(0, 256, 3, dtype=np.uint8)
    elif content == "thin_stripes":  # many runs inside every window
        for y in range(0, h, 3):
            img[y, 200:700] = rng.integers(0, 256, 3, dtype=np.uint8)
        for x in range(800, 1100, 2):
            img[:, x] = rng.integers(0, 256, 3, dtype=np.uint8)
    else:  # corners: small rectangles, several per band
        for _ in range(120):
            y0, x0 = int(rng.integers(0, h - 4)), int(rng.integers(0, w - 4))
            img[y0:y0 + int(rng.integers(2, 40)), x0:x0 + int(rng.integers(2, 60))] = \
                rng.integers(0, 256, 3, dtype=np.uint8)
    for r, L in ((10, 256), (8, 255), (15, 40), (3, 100)):
        want = oracle_lib.oracle_filter(img, r, L, 0, threads=4)
        assert np.array_equal(run(gpu, img, r, L, 0, SLIDE, L == 256), want), (content, r, L)


def test_slide_wide_image_long_flat_stretches(gpu):
    """Passes thousands of columns wide: several jumps over flat stretches per
    pass (the lookahead covers 1024 columns), edges right after a jump, at the
    ends of the lookahead window and in the last columns."""
    rng = np.random.default_rng(11)
    h, w = 96, 16384 + 17
    img = np.empty((h, w, 3), np.uint8)
    img[:] = rng.integers(0, 256, 3, dtype=np.uint8)
    for x in (63, 64, 65, 1023, 1024, 1025, 1087, 2047, 2048, 5000, 5001, 9000, 12287, 12288, w - 12, w - 1):
        img[:, x:] = rng.integers(0, 256, 3, dtype=np.uint8)
    img[40:50, 3000:11000] = rng.integers(0, 256, 3, dtype=np.uint8)
    img[70:, 7000:7003] = rng.integers(0, 256, 3, dtype=np.uint8)
    for r, L in ((10, 256), (8, 64), (15, 255)):
        want = oracle_lib.oracle_filter(img, r, L, 0, threads=8)
        assert np.array_equal(run(gpu, img, r, L, 0, SLIDE, L == 256), want), (r, L)


def test_slide_more_bands_than_the_plan_orders(gpu):
    """The work plan orders up to 1024 bands by cost; a taller launch keeps
    the natural order (identity permutation)."""
    rng = np.random.default_rng(5)
    h, w = 33000, 48  # 1031 bands of 32 rows
    img = np.empty((h, w, 3), np.uint8)
    img[:] = rng.integers(0, 256, 3, dtype=np.uint8)
    for _ in range(300):
        y0, x0 = int(rng.integers(0, h - 4)), int(rng.integers(0, w - 4))
        img[y0:y0 + int(rng.integers(2, 400)), x0:x0 + int(rng.integers(2, 30))] = \
            rng.integers(0, 256, 3, dtype=np.uint8)
    want = oracle_lib.oracle_filter(img, 3, 100, 0, threads=8)
    assert np.array_equal(run(gpu, img, 3, 100, 0, SLIDE), want)


@pytest.mark.parametrize("content", ["flat", "smooth", "two_tone", "white"])
def test_skew_tie_heavy_content(gpu, content):
    """Smooth / flat content: single-bin windows, many exact ties, bin L (white)."""
    rng = np.random.default_rng(7)
    h, w = 97, 211
    if content == "flat":
        img = np.full((h, w, 3), 77, np.uint8)
    elif content == "smooth":
        base = rng.integers(0, 256, 3)
        img = np.clip(base + rng.integers(-10, 11, (h, w, 3)), 0, 255).astype(np.uint8)
    elif content == "two_tone":
        img = np.where(rng.random((h, w, 1)) < 0.5, 40, 200).astype(np.uint8).repeat(3, 2)
    else:
        img = np.where(rng.random((h, w, 1)) < 0.5, 255, 254).astype(np.uint8).repeat(3, 2)
    for r, L in ((3, 20), (7, 30), (15, 20), (2, 1)):
        want = oracle_lib.oracle_filter(img, r, L, 0, threads=4)
        assert np.array_equal(run(gpu, img, r, L, 0, SKEW), want), (content, r, L)
        assert np.array_equal(run(gpu, img, r, L, 0, DIRECT), want), (content, r, L)
        if column_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, 0, COLUMN), want), (content, r, L)
        if planes_ok(r, L):
            assert np.array_equal(run(gpu, img, r, L, 0, PLANES), want), (content, r, L)


@pytest.mark.parametrize("L", [23, 30, 31])
def test_skew_bin_groups_on_smooth_batches(gpu, L):
    """KEY launches with >= 24 bins skip the bin groups a phase never sees
    (block bin masks from the shear pre-pass): smooth ramps whose bin range
    drifts across the frame and between frames, odd sizes, partial bands."""
    rng = np.random.default_rng(L)
    for (w, h, f) in ((333, 97, 3), (130, 517, 2), (1000, 40, 2)):
        yy, xx = np.mgrid[0:h, 0:w]
        frames = []
        for k in range(f):
            base = (xx * (2 + k) + yy * (3 - k)) % 256
            img = np.stack([base, (base + 40 * k) % 256, (255 - base)], axis=-1)
            img = np.clip(img + rng.integers(-6, 7, img.shape), 0, 255).astype(np.uint8)
            frames.append(img)
        batch = np.stack(frames)
        torch = pytest.importorskip("torch")
        dev_in = torch.from_numpy(batch).cuda()
        dev_out = torch.empty_like(dev_in)
        for r in (3, 7):
            got = gpu.apply_cuda_batch(batch, gpu.FilterParams(r, L), gpu.CudaConfig(kernel=SKEW))
            # one launch over all frames (the per-frame bin-mask tables)
            gpu.apply_cuda_device(dev_in.data_ptr(), dev_out.data_ptr(), w, h, gpu.FilterParams(r, L),
                                  gpu.CudaConfig(device=0, kernel=SKEW), frames=f)
            torch.cuda.synchronize()
            dgot = dev_out.cpu().numpy()
            for k in range(f):
                want = oracle_lib.oracle_filter(batch[k], r, L, 0, threads=4)
                assert np.array_equal(got[k], want), (w, h, k, r, L)
                assert np.array_equal(dgot[k], want), (w, h, k, r, L, "device batch")


def test_large_radius_and_l256(gpu):
    rng = np.random.default_rng(9)
    for r, L in ((16, 20), (20, 5), (31, 255), (12, 256), (3, 256)):
        h, w = 2 * r + 1 + 17, 2 * r + 1 + 29
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        want = oracle_lib.oracle_filter(img, r, L, 1)
        assert np.array_equal(run(gpu, img, r, L, 1, AUTO, L == 256), want), (r, L)


def test_edge_shapes(gpu):
    rng = np.random.default_rng(11)
    img = np.array([[[42, 43, 44]]], np.uint8)  # test_parallel.cpp:142-145
    for b in (0, 1):
        assert np.array_equal(run(gpu, img, 0, 20, b), img)
    for (h, w, r) in ((5, 9, 0), (3, 1000, 1), (1000, 3, 1), (31, 31, 15), (33, 257, 15),
                      (64, 129, 15), (40, 1, 0), (2, 2, 0)):
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        for L in (1, 20, 255):
            for b in (0, 1):
                want = oracle_lib.oracle_filter(img, r, L, b)
                assert np.array_equal(run(gpu, img, r, L, b), want), (h, w, r, L, b)


def test_identity_uniform_and_border_policy(gpu):
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (5, 9, 3), dtype=np.uint8)
    for b in (0, 1):  # test_filter.cpp:192-198: r=0 is the identity
        assert np.array_equal(run(gpu, img, 0, 20, b), img)
    uni = np.empty((9, 12, 3), np.uint8)
    uni[:] = (17, 170, 71)  # test_filter.cpp:200-203
    assert np.array_equal(run(gpu, uni, 2, 20, 0), uni)
    img = rng.integers(0, 256, (8, 10, 3), dtype=np.uint8)  # test_filter.cpp:213-233
    z, c = run(gpu, img, 2, 20, 1), run(gpu, img, 2, 20, 0)
    inner = np.zeros((8, 10), bool)
    inner[2:6, 2:8] = True
    assert np.array_equal(z[inner], c[inner])
    assert (z[~inner] == 0).all() and np.array_equal(c[~inner], img[~inner])


def test_output_within_neighbourhood_extremes(gpu):
    rng = np.random.default_rng(5)  # test_filter.cpp:235-266
    for _ in range(20):
        h, w = int(rng.integers(3, 40)), int(rng.integers(3, 40))
        r = int(rng.integers(1, max(1, min(3, (min(h, w) - 1) // 2)) + 1))
        L = int(rng.integers(1, 256))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        out = run(gpu, img, r, L)
        for y in range(r, h - r):
            for x in range(r, w - r):
                win = img[y - r:y + r + 1, x - r:x + r + 1].reshape(-1, 3)
                assert (out[y, x] >= win.min(0)).all() and (out[y, x] <= win.max(0)).all()


def test_validation_errors(gpu):
    img = np.zeros((8, 8, 3), np.uint8)  # test_filter.cpp:293-304
    P = gpu.FilterParams
    for p in (P(4, 20), P(-1, 20), P(1, 0), P(1, 256)):
        with pytest.raises(gpu.InvalidArgument):
            gpu.apply_cuda(img, p)
    gpu.apply_cuda(np.zeros((1, 1, 3), np.uint8), P(0, 20))
    gpu.apply_cuda(img, P(3, 20))
    with pytest.raises(gpu.InvalidArgument, match="intensity_levels must be in"):
        gpu.apply_cuda(img, P(1, 257), gpu.CudaConfig(allow_levels_256=True))
    with pytest.raises(gpu.InvalidArgument):  # forcing SKEW beyond its r <= 15 range
        gpu.apply_cuda(np.zeros((40, 40, 3), np.uint8), P(16, 20), gpu.CudaConfig(kernel=SKEW))


def test_bands_reassemble_whole_image(gpu):
    """Row bands with r-row halos (multi-GPU partition) == whole-image result,
    every output row covered exactly once (test_parallel.cpp:65-103 analogue)."""
    rng = np.random.default_rng(12)
    h, w = 301, 173
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    for r, L, b in ((15, 20, 0), (7, 30, 1), (2, 255, 0), (0, 20, 1)):
        whole = run(gpu, img, r, L, b)
        assert np.array_equal(whole, oracle_lib.oracle_filter(img, r, L, b, threads=4))
        for n in (1, 2, 3, 8, 13):
            cuts = [h * k // n for k in range(n + 1)]
            parts = []
            for y0, y1 in zip(cuts[:-1], cuts[1:]):
                lo, hi = gpu.band_input_rows(h, y0, y1, r)
                parts.append(gpu.apply_cuda_band(img[lo:hi], h, y0, y1,
                                                 gpu.FilterParams(r, L, gpu.BorderPolicy(b))))
            assert sum(p.shape[0] for p in parts) == h
            assert np.array_equal(np.concatenate(parts), whole), (r, L, b, n)


def test_batch_equals_per_frame(gpu):
    rng = np.random.default_rng(13)
    frames = rng.integers(0, 256, (5, 67, 91, 3), dtype=np.uint8)
    p = gpu.FilterParams(7, 30)
    out = gpu.apply_cuda_batch(frames, p)
    for f in range(5):
        assert np.array_equal(out[f], oracle_lib.oracle_filter(frames[f], 7, 30))


def test_batch_beyond_grid_z_limit(gpu):
    """More frames than gridDim.z allows (65535): consecutive launches."""
    rng = np.random.default_rng(77)
    n = 65535 + 1200
    frames = rng.integers(0, 256, (n, 4, 5, 3), dtype=np.uint8)
    torch = pytest.importorskip("torch")
    dev_in = torch.from_numpy(frames).cuda()
    for k in (AUTO, SKEW, DIRECT):
        got = gpu.apply_cuda_batch(frames, gpu.FilterParams(1, 20), gpu.CudaConfig(kernel=k))
        dev_out = torch.empty_like(dev_in)
        gpu.apply_cuda_device(dev_in.data_ptr(), dev_out.data_ptr(), 5, 4, gpu.FilterParams(1, 20),
                              gpu.CudaConfig(device=0, kernel=k), frames=n)
        torch.cuda.synchronize()
        dgot = dev_out.cpu().numpy()
        for i in (0, 1, 65534, 65535, 65536, n - 1):
            want = oracle_lib.oracle_filter(frames[i], 1, 20)
            assert np.array_equal(got[i], want), (k, i)
            assert np.array_equal(dgot[i], want), (k, i, "device")


def test_device_pointer_path_with_torch_stream(gpu):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(14)
    img = rng.integers(0, 256, (130, 250, 3), dtype=np.uint8)
    want = oracle_lib.oracle_filter(img, 15, 20)
    dev_in = torch.from_numpy(img).cuda()
    dev_out = torch.empty_like(dev_in)
    stream = torch.cuda.Stream()
    cfg = gpu.CudaConfig(device=dev_in.device.index, stream=stream.cuda_stream)
    with torch.cuda.stream(stream):
        gpu.apply_cuda_device(dev_in.data_ptr(), dev_out.data_ptr(), 250, 130,
                              gpu.FilterParams(15, 20), cfg)
    stream.synchronize()
    assert np.array_equal(dev_out.cpu().numpy(), want)


def test_launch_counter_advances(gpu):
    before = gpu.kernel_launches()
    run(gpu, np.zeros((40, 40, 3), np.uint8), 3, 20)
    assert gpu.kernel_launches() >= before + 1  # direct tile kernel (border blocks fused)


@pytest.mark.parametrize("kernel", [AUTO, DIRECT, SKEW, SLIDE, COLUMN, PLANES])
@pytest.mark.parametrize("r", [3, 6])
@pytest.mark.parametrize("in_off,out_off", [(0, 0), (1, 3), (5, 2), (16, 7)])
def test_device_pointers_at_unaligned_offsets(gpu, kernel, r, in_off, out_off):
    """The fused border job copies 16 bytes per store: unaligned and mutually
    misaligned device pointers take its head / byte-assembling paths.  Bytes
    around the output stay untouched."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(in_off * 31 + out_off)
    w, h, L = 203, 77, 20
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    n = img.size
    for b in (0, 1):
        want = oracle_lib.oracle_filter(img, r, L, b)
        dev_in = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
        dev_in[in_off:in_off + n] = torch.from_numpy(img.reshape(-1)).cuda()
        dev_out = torch.full((n + 64,), 0xCD, dtype=torch.uint8, device="cuda")
        cfg = gpu.CudaConfig(device=0, kernel=kernel)
        gpu.apply_cuda_device(dev_in.data_ptr() + in_off, dev_out.data_ptr() + out_off, w, h,
                              gpu.FilterParams(r, L, gpu.BorderPolicy(b)), cfg)
        torch.cuda.synchronize()
        got = dev_out.cpu().numpy()
        assert np.array_equal(got[out_off:out_off + n].reshape(h, w, 3), want), (b, kernel)
        assert (got[:out_off] == 0xCD).all() and (got[out_off + n:] == 0xCD).all()


@pytest.mark.parametrize("r,L", [(1, 31), (4, 20), (7, 30)])
def test_planes_multi_round_batch(gpu, r, L):
    """A launch of several rounds of blocks takes the bit-plane family's
    block-shared column sums (one array per block, block barriers per row):
    a 48-frame batch against the oracle on sampled frames and the per-frame
    calls on all of them; 16-column-multiple width (TMA tile loads) and a
    ragged one (LDG tile loads)."""
    rng = np.random.default_rng(r * 100 + L)
    for w in (608, 601):
        h, f = 301, 48
        frames = rng.integers(0, 256, (f, h, w, 3), dtype=np.uint8)
        p = gpu.FilterParams(r, L)
        c = gpu.CudaConfig(kernel=PLANES)
        out = gpu.apply_cuda_batch(frames, p, c)
        for i in (0, 17, f - 1):
            assert np.array_equal(out[i], oracle_lib.oracle_filter(frames[i], r, L, 0, threads=8)), (w, i)
        for i in range(f):
            assert np.array_equal(out[i], gpu.apply_cuda(frames[i], p, c)), (w, i)


@pytest.mark.parametrize("y0,y1", [(0, 97), (40, 233), (230, 301)])
def test_planes_bands(gpu, y0, y1):
    """Row bands (the multi-GPU unit) through the bit-plane family: the band
    input starts at in_row0 > 0 (the TMA box's row coordinate is relative to
    it) and ends inside the image."""
    rng = np.random.default_rng(y0 + y1)
    img = rng.integers(0, 256, (301, 640, 3), dtype=np.uint8)
    for r in (2, 5, 7):
        p = gpu.FilterParams(r, 20)
        c = gpu.CudaConfig(kernel=PLANES)
        whole = oracle_lib.oracle_filter(img, r, 20, 0, threads=8)
        lo, hi = gpu.band_input_rows(301, y0, y1, r)
        band = gpu.apply_cuda_band(img[lo:hi], 301, y0, y1, p, c)
        assert np.array_equal(band, whole[y0:y1]), (r, y0, y1)


@pytest.mark.parametrize("w,h", [(16, 16), (16, 300), (32, 7), (48, 129), (160, 15), (2048, 31)])
def test_planes_tma_edge_shapes(gpu, w, h):
    """Widths that are multiples of 16 take the TMA tile path: boxes wider
    and taller than the tensor (zero-filled), a single 128-column block, and
    images only 2r+1 rows high."""
    rng = np.random.default_rng(w * 1000 + h)
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    for r in (1, 3, 7):
        if min(w, h) < 2 * r + 1:
            continue
        for L in (20, 31):
            want = oracle_lib.oracle_filter(img, r, L, 0, threads=4)
            assert np.array_equal(run(gpu, img, r, L, 0, PLANES), want), (w, h, r, L)
