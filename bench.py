#!/usr/bin/env python3
"""Benchmark of the B200 oil-paint filter hot path (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl b200|reference]

Workload (config.workload): BASELINE.json's large-radius configuration, the one
the north-star target is quoted on -- config 4, 16384x16384 uniform-noise RGB8,
r=15, L=20, CopyInput (the other four configs are parity-test cases;
--config selects them for manual runs).  A "step" is one pass of the filter over
the whole image.  N>1: one process per GPU (under torchrun, or -- when
WORLD_SIZE is unset -- bench.py re-launches itself under torch.distributed.run
with N ranks); the image's rows are split into N contiguous bands with r-row
halos, every rank generates and filters only its own band; no
collective on the data path (NCCL is used only for the barrier, the
max-over-ranks timing and the per-rank report).

Reported:
  value     output MP/s of the whole job, device-resident inputs, timed with CUDA
            events on the launching stream, max over ranks; the 805 MB input is
            larger than the 126 MB L2, so no flush is needed between steps.
  e2e       the same metric through the C-ABI host-pointer call (pinned host
            buffers, H2D + kernels + D2H inside the timed region).
  roofline  issue-rate bound: colhist model ops/px x interior
            pixels / kernel time vs 148 SMs x 4 warp-instr/clk x 32 lanes x
            1965 MHz; the HBM side (6 B/px at 6548.5 GB/s measured) is reported
            beside it.
  cpu_baseline  the unmodified reference library (oracle/_ref, apply_parallel's
            row-band engine) on all host cores of the box, on a bounded band of
            the same image (rank 0's band; every N, every config).

--impl reference: the reference's own CPU engine on the same workload, metric
and config (rank 0 only).  That arm loads only oracle/_ref (the reference
library built from its sources, plus the harness generators of configs 2/3/5):
it never imports paper_1405_1020_b200 or maps liboilpaint_b200.so; the
workload table is read from paper_1405_1020_b200/workloads.py by file path.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "output megapixels/sec at radius r, levels L (1/2/4/8 B200) and % of roofline"


def load_workloads() -> dict:
    """paper_1405_1020_b200/workloads.py by file path (plain data: no package
    import, no library load)."""
    name = "_opc_workloads"
    if name not in sys.modules:
        spec = importlib.util.spec_from_file_location(
            name, ROOT / "paper_1405_1020_b200" / "workloads.py")
        mod = importlib.util.module_from_spec(spec)
        sys.modules[name] = mod
        spec.loader.exec_module(mod)
    return sys.modules[name].WORKLOADS


PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}


def load_peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return dict(PEAKS_FALLBACK), "fallback"


def colhist_ops_per_px(bins: int) -> int:
    # colhist (Perreault-Hebert, O(B)) = 7*2 + 8*B + 3*B + 12 lane-ops
    return 7 * 2 + 8 * bins + 3 * bins + 12


def best_fit_model(radius: int, bins: int) -> tuple[str, int]:
    """The cheapest of SURVEY.md 8(d)'s per-pixel op models (the highest,
    i.e. most conservative, roof): direct 7n^2 + 4B + 12, slide (Huang)
    7*2n + 3B + 12, colhist 7*2 + 11B + 12, n = 2r + 1."""
    n = 2 * radius + 1
    models = {"direct": 7 * n * n + 4 * bins + 12, "slide": 7 * 2 * n + 3 * bins + 12,
              "colhist": colhist_ops_per_px(bins)}
    name = min(models, key=models.get)
    return name, models[name]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons, sampled every 20 ms from before the
    warm-up to after the timed region; summary() keeps the samples whose
    timestamps fall inside the timed region [mark_start(), mark_end()]."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.3)  # let the sampler start before the measured region
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self._t.join(timeout=2)

    def summary(self) -> dict:
        mhz, max_mhz, reasons, power = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, ln in self.lines:
            # the line arrives <= 20 ms after it was sampled
            if self.t0 is not None and not (self.t0 <= t <= self.t1 + 0.04):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 10:
                continue
            try:
                mhz.append(float(f[2]))
                max_mhz = max(max_mhz, float(f[3]))
                power.append(float(f[4]))
            except ValueError:
                continue
            for name, v in zip(names, f[6:10]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(mhz) if mhz else None,
                "sm_max_mhz": max_mhz or None, "reasons": sorted(reasons),
                "samples": len(mhz), "power_w_max": max(power) if power else None}


# ----------------------------------------------------------------------------
# CPU legs (TEST INFRASTRUCTURE as the checker / baseline): the reference
# library (oracle/_ref) or, if it was not built, the C restatement (oracle/).
# Used only for cpu_baseline and --impl reference.
# ----------------------------------------------------------------------------

def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuEngine:
    """The reference engine body (parallel_for_rows + filter_pixel, the engine
    of apply_parallel, proj/src/parallel.cpp:110-132) from oracle/_ref, or the
    oracle's C port when oracle/_ref is absent."""

    def __init__(self):
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_lib
        self.kind = "reference"
        try:
            self.ref = oracle_lib.load_ref()
        except (FileNotFoundError, OSError):
            self.ref = None
            self.kind = "port"
            self.oracle = oracle_lib.oracle()

    def generate_rows(self, wl, nrows: int, frame: int = 0) -> np.ndarray:
        """Rows [0, nrows) of the workload's input (frame `frame`): the
        reference generator (proj/src/pattern.cpp:64-76, Noise{seed}) for the
        noise configs, the harness generators in oracle/_ref for the others."""
        out = np.empty((nrows, wl.width, 3), np.uint8)
        if wl.pattern == 0:
            # Noise: byte i = byte (i mod 8) of stream word i / 8 -- the first
            # nrows rows of the W x H image are the W x nrows image
            if self.ref is not None:
                rc = self.ref.ref_generate(0, wl.seed, wl.width, nrows, out.ctypes.data)
                assert rc == 0, self.ref.ref_last_error()
            else:
                self.oracle.oracle_noise(wl.seed, out.ctypes.data, out.size)
            return out
        if self.ref is None:
            raise RuntimeError(f"{wl.name}: its generator lives in oracle/_ref, which is not built")
        rc = self.ref.ref_harness_generate_rows(wl.pattern, wl.seed, wl.width, wl.height, frame, 0,
                                                nrows, out.ctypes.data, 0)
        assert rc == 0
        return out

    def band(self, img: np.ndarray, out: np.ndarray, radius: int, levels: int, y0: int, y1: int,
             threads: int) -> None:
        """Interior rows [y0, y1) of the image `img` (all of whose rows are
        given) into the same rows of `out`."""
        h, w, _ = img.shape
        if self.ref is not None:
            rc = self.ref.ref_filter_band(img.ctypes.data, out.ctypes.data, w, h, radius, levels,
                                          y0, y1, threads)
            assert rc == 0
        else:  # C port: filter a sub-image holding the band plus halos
            sub = np.ascontiguousarray(img[y0 - radius:y1 + radius])
            tmp = np.empty_like(sub)
            rc = self.oracle.oracle_filter_mt(sub.ctypes.data, tmp.ctypes.data, w, sub.shape[0],
                                              radius, levels, 0, threads)
            assert rc == 0
            out[y0:y1] = tmp[radius:radius + (y1 - y0)]


class CpuSample:
    """A bounded sample of the workload for the CPU engine: interior rows
    [r, r + rows) of an image whose first rows are `src` (a rank's band, or
    rows generated by CpuEngine), full width -- rows chosen so one run takes
    about target_s on `threads` threads."""

    def __init__(self, eng: CpuEngine, wl, threads: int, target_s: float, src=None):
        self.eng, self.wl, self.threads = eng, wl, threads
        r = wl.radius
        self.max_rows = (src.shape[0] if src is not None else wl.height) - 2 * r
        self.src = src
        rows = max(1, min(self.max_rows, 4 * threads))
        while True:
            t = time.perf_counter()
            self._run(rows)
            dt = time.perf_counter() - t
            if dt >= 0.5 or rows >= self.max_rows:
                break
            rows = min(self.max_rows, rows * 4)
        rate = rows / max(dt, 1e-6)
        self.rows = int(max(1, min(self.max_rows, rate * target_s)))
        self._image(self.rows)

    def _image(self, rows: int) -> np.ndarray:
        need = rows + 2 * self.wl.radius
        if self.src is None or self.src.shape[0] < need:
            self.src = self.eng.generate_rows(self.wl, min(self.wl.height, max(need, 64)))
            self.out = np.zeros_like(self.src)
        elif not hasattr(self, "out") or self.out.shape != self.src.shape:
            self.out = np.zeros_like(self.src)
        return self.src

    def _run(self, rows: int) -> None:
        img = self._image(rows)
        r = self.wl.radius
        self.eng.band(img, self.out, r, self.wl.levels, r, r + rows, self.threads)

    def run(self) -> float:
        t = time.perf_counter()
        self._run(self.rows)
        return time.perf_counter() - t

    @property
    def megapixels(self) -> float:
        return self.rows * self.wl.width / 1e6  # output MP: rows x full width

    def describe(self, seconds: float) -> str:
        r = self.wl.radius
        what = ("reference apply_parallel row-band engine (parallel_for_rows + filter_pixel)"
                if self.eng.kind == "reference" else "C port of the reference engine")
        frame = " (frame 0)" if self.wl.frames > 1 else ""
        return (f"rows [{r}, {r + self.rows}) x {self.wl.width} cols of the {self.wl.name} "
                f"image{frame} per run ({self.megapixels:.2f} MP, {seconds:.2f} s), {what}, "
                f"{self.threads} threads, {cpu_model()}")


def workload_config(wl, n: int) -> dict:
    return {"workload": f"{wl.name}: {wl.description}", "width": wl.width,
            "height": wl.height, "frames": wl.frames, "radius": wl.radius,
            "levels": wl.levels, "border": "CopyInput", "partition":
            ("frames" if wl.frames > 1 else "row bands with r-row halos") + f" over {n} GPU(s)",
            "l2": l2_note(rank0_in_bytes(wl, n))}


def rank0_in_bytes(wl, n: int) -> int:
    """Input bytes of rank 0 of an n-GPU run (its row band plus halos, or its frames)."""
    W, H, F = wl.width, wl.height, wl.frames
    if F == 1:
        y1 = H // n
        return (min(H, y1 + wl.radius) - 0) * W * 3
    return (F // n) * H * W * 3


def l2_note(in_bytes: int) -> str:
    """Per-rank input bytes vs the L2 (main() flushes below 2 x 126 MiB)."""
    mb = in_bytes / 2**20
    if mb >= 2 * 126:
        return f"input {mb:.0f} MiB per GPU > 126 MB L2 (no flush needed)"
    return f"input {mb:.1f} MiB per GPU < 2 x 126 MB L2: L2 flushed between timed steps (512 MiB memset, untimed)"


def reference_arm(args, wl) -> None:
    """--impl reference: the reference's own engine on the host cores, rank 0
    only; loads oracle/_ref and nothing of the product."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = host_threads()
    # each step a bounded sample; the whole run stays within about 2 minutes
    step_s = float(os.environ.get("OILPAINT_REF_STEP_S",
                                  min(4.0, 120.0 / max(1, args.steps + args.warmup))))
    eng = CpuEngine()
    sample = CpuSample(eng, wl, threads, step_s)
    for _ in range(args.warmup):
        sample.run()
    times = [sample.run() for _ in range(args.steps)]
    total = sum(times)
    value = sample.megapixels * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "MP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * total / len(times), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(wl, args.gpus),
        "cpu_baseline": {"value": round(value, 4), "unit": "MP/s", "cores": threads,
                         "kind": eng.kind, "sample": sample.describe(total / len(times))},
        "e2e": {"value": round(value, 4), "unit": "MP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 without a torchrun environment: run this script as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")

    wl = load_workloads()[args.config]
    if args.impl == "reference":
        reference_arm(args, wl)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    run_b200(args, wl)


def run_b200(args, wl) -> None:
    import torch
    import torch.distributed as dist
    import paper_1405_1020_b200 as opc
    from paper_1405_1020_b200 import _lib

    cfg = opc.CONFIGS[wl.name]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: one process per "
                         "GPU is required (launch with --nproc-per-node equal to --gpus)")
    # One process per GPU over NCCL.  OPC_BENCH_BACKEND=gloo with more ranks
    # than GPUs is a plumbing check only (ranks share devices; not a number
    # to report): the rank -> device map wraps around.
    backend = os.environ.get("OPC_BENCH_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    if backend == "nccl" and world > ndev:
        raise SystemExit(f"bench.py: {world} ranks but {ndev} visible GPU(s)")
    if backend != "nccl":
        local = local % ndev
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            # the communicator log (rank -> device, transport) goes to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    W, H, F = cfg.width, cfg.height, cfg.frames
    r, L = cfg.radius, cfg.levels
    params = opc.FilterParams(r, L, opc.BorderPolicy.CopyInput)
    stream = torch.cuda.Stream()
    ccfg = opc.CudaConfig(device=local, stream=stream.cuda_stream,
                          allow_levels_256=(L == 256))

    # ---- this rank's share: row band (single image) or frames (batch); each
    # rank generates only its own input rows / frames ----
    if F == 1:
        y0, y1 = opc.band_begin(H, world, rank), opc.band_begin(H, world, rank + 1)
        lo, hi = opc.band_input_rows(H, y0, y1, r)
        host_in = torch.empty((hi - lo, W, 3), dtype=torch.uint8).pin_memory()
        cfg.generate_rows(lo, hi - lo, out=host_in.numpy())
        out_shape = (y1 - y0, W, 3)
        my_frames = 1
        out_pixels = (y1 - y0) * W
        interior = max(0, min(y1, H - r) - max(y0, r)) * (W - 2 * r)
        share = {"rows": [y0, y1], "input_rows": [lo, hi]}
    else:
        f0, f1 = opc.band_begin(F, world, rank), opc.band_begin(F, world, rank + 1)
        my_frames = f1 - f0
        host_in = torch.empty((my_frames, H, W, 3), dtype=torch.uint8).pin_memory()
        for i in range(my_frames):
            cfg.generate(f0 + i, out=host_in[i].numpy())
        out_shape = (my_frames, H, W, 3)
        out_pixels = my_frames * H * W
        interior = my_frames * (H - 2 * r) * (W - 2 * r)
        share = {"frames": [f0, f1]}
    dev_in = host_in.to(f"cuda:{local}")
    dev_out = torch.empty(out_shape, dtype=torch.uint8, device=f"cuda:{local}")

    def step_device():
        if F == 1:
            opc.apply_cuda_band_device(dev_in.data_ptr(), dev_out.data_ptr(), W, H, y0, y1,
                                       params, ccfg)
        else:
            opc.apply_cuda_device(dev_in.data_ptr(), dev_out.data_ptr(), W, H, params, ccfg,
                                  frames=my_frames)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step_device()
    stream.synchronize()

    # Inputs smaller than twice the 126 MB L2 (configs 1-3, and the bands of a
    # wide split): the L2 is flushed between timed steps (a 512 MB memset on
    # the stream, outside the steps' event pairs), so every step reads its
    # input from HBM.
    flush = None
    if host_in.numel() < 2 * 126 * 2**20:
        flush = torch.empty(512 * 2**20, dtype=torch.uint8, device=f"cuda:{local}")
    def timed_pass():
        """K steps between CUDA events on the launch stream (L2 flushed
        outside each step's event pair when needed); per-step ms."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        ev_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        with torch.cuda.stream(stream):
            if flush is None:
                ev[0].record(stream)
                for i in range(args.steps):
                    step_device()
                    ev[i + 1].record(stream)
            else:
                for i in range(args.steps):
                    flush.zero_()
                    ev[i].record(stream)
                    step_device()
                    ev_end[i].record(stream)
        stream.synchronize()
        if flush is None:
            return [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)], ev[0].elapsed_time(ev[args.steps])
        ms = [ev[i].elapsed_time(ev_end[i]) for i in range(args.steps)]
        return ms, sum(ms)

    launches0 = opc.kernel_launches()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        clocks.mark_start()
        step_ms, my_total_ms = timed_pass()
        clocks.mark_end()
    torch.cuda.synchronize()
    barrier()
    launches = opc.kernel_launches() - launches0
    # Live per-kernel timing for the roofline: a second K-step pass in which
    # the library brackets each of its kernel launches with CUDA events on the
    # launch stream (opc_kernel_timing).  Those extra events cost ~5-7 us of
    # stream time per step (scripts/step_gap.py), so `value` comes from the
    # pass above, without them.
    opc.kernel_timing(True)
    hook_step_ms, _ = timed_pass()
    family = opc.plan_kernel(W, H, r, L, my_frames)  # OPC_KERNEL_DIRECT/SKEW/SLIDE/COLUMN/PLANES = 1-5
    # timing ids: 1-3 as the families, 6 column, 7 planes
    kid = {4: _lib.OPC_KID_COLUMN, 5: _lib.OPC_KID_PLANES}.get(family, family)
    kernel_total_ms, kernel_n = opc.kernel_timing_read(kid)
    pre_ms, _ = opc.kernel_timing_read(_lib.OPC_KID_PREPASS)
    border_ms, _ = opc.kernel_timing_read(_lib.OPC_KID_BORDER)
    opc.kernel_timing(False)
    red_dev = f"cuda:{local}" if backend == "nccl" else "cpu"
    t = torch.tensor([my_total_ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    job_pixels = F * W * H
    value = job_pixels / (ms_per_step / 1e3) / 1e6

    # ---- end to end through the public C-ABI with host buffers ----
    import ctypes as _ct
    from paper_1405_1020_b200._lib import LIB
    host_out = torch.empty(out_shape, dtype=torch.uint8).pin_memory()
    c_e2e = opc.CudaConfig(device=local, allow_levels_256=(L == 256)).to_c()

    def step_e2e(src, dst):
        if F == 1:
            rc = LIB.opc_filter_rgb8_band(src.ctypes.data, dst.ctypes.data, W, H, y0, y1,
                                          r, L, 0, _ct.byref(c_e2e))
        else:
            rc = LIB.opc_filter_rgb8_batch(src.ctypes.data, dst.ctypes.data, my_frames, W,
                                           H, r, L, 0, _ct.byref(c_e2e))
        assert rc == 0, LIB.opc_last_error()

    e2e_step_ms: list[float] = []  # this rank's wall time of every timed pinned-buffer call

    def time_e2e(src, dst, record=None) -> float:
        step_e2e(src, dst)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            step_e2e(src, dst)
            if record is not None:
                record.append(round((time.perf_counter() - t1) * 1e3, 4))
        dt = time.perf_counter() - t0
        te = torch.tensor([dt], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return job_pixels * args.e2e_steps / float(te.item()) / 1e6

    e2e_value = time_e2e(host_in.numpy(), host_out.numpy(), e2e_step_ms)
    # the e2e output must equal the device-resident output
    assert torch.equal(host_out, dev_out.cpu()), "e2e output differs from device output"
    # the same call from pageable buffers (a std::vector Image / numpy array):
    # staged through the library's pinned ring
    page_in = np.array(host_in.numpy(), copy=True)
    page_out = np.empty(out_shape, np.uint8)
    e2e_pageable = time_e2e(page_in, page_out)
    assert np.array_equal(page_out, host_out.numpy()), "pageable e2e output differs"
    del page_in, page_out

    # ---- roofline (issue-rate bound) ----
    peaks, peaks_kind = load_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    num_sms = torch.cuda.get_device_properties(local).multi_processor_count
    peak_ops = num_sms * 4 * 32 * sm_mhz * 1e6
    model_name, ops_px = best_fit_model(r, L + 1)
    # achieved = algorithmic lane-ops of the timed steps / time inside the
    # dominant kernel (its launches, CUDA events on the launch stream)
    kernel_ms = kernel_total_ms / max(1, kernel_n)
    ops_per_step = ops_px * interior
    model_label = (f"{model_name} {ops_px} lane-ops per interior pixel (SURVEY 8d best fit, "
                   f"B={L + 1})")
    executed = None
    if family == 3:
        # The slide family adapts to the content (flat steps skip their
        # updates, the argmax rescans only when the winner may have changed),
        # so a per-pixel model overstates its work.  Its op count is what one
        # counting launch of the same step on the same input executed
        # (OPC_FLAG_COUNT_OPS, outside the timed region), priced with SURVEY
        # 8(d)'s primitive costs.
        cnt_cfg = opc.CudaConfig(device=local, stream=stream.cuda_stream,
                                 allow_levels_256=(L == 256), count_ops=True)
        opc.op_counts(local, reset=True)
        with torch.cuda.stream(stream):
            if F == 1:
                opc.apply_cuda_band_device(dev_in.data_ptr(), dev_out.data_ptr(), W, H, y0, y1,
                                           params, cnt_cfg)
            else:
                opc.apply_cuda_device(dev_in.data_ptr(), dev_out.data_ptr(), W, H, params,
                                      cnt_cfg, frames=my_frames)
        stream.synchronize()
        executed = opc.op_counts(local, reset=True)
        ops_per_step = (12 * executed["pixels"] + 3 * executed["steps"] +
                        7 * executed["updates"] + 3 * executed["bins_examined"] +
                        7 * executed["sum_pixels"])
        model_label = ("slide, executed primitives of one counted launch (OPC_FLAG_COUNT_OPS): "
                       "12 x pixels + 3 x lane-steps + 7 x count updates + 3 x bins examined "
                       "by rescans + 7 x window pixels summed on winner changes (SURVEY 8d "
                       f"costs); the best-fit per-pixel model ({model_name} {ops_px}/px) would "
                       f"be {ops_px * interior} per launch")
    achieved_ops = ops_per_step * args.steps / (kernel_total_ms / 1e3)
    step_total_ms = sum(step_ms)
    traffic = None
    tp = ROOT / "profiles" / f"{cfg.name}_dram_bytes.json"
    if tp.exists() and world == 1:
        traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")
    hbm_gbs = float(peaks.get("hbm_gbs", 6650.0))
    alg_bytes = 6 * out_pixels
    roofline = {
        "bound": "issue", "achieved": round(achieved_ops / 1e12, 3),
        "peak": round(peak_ops / 1e12, 3), "unit": "Tlane-op/s",
        "frac": round(achieved_ops / peak_ops, 4), "traffic": traffic,
        "model": f"{model_label}; "
                 f"{num_sms} SMs x 4 x 32 x {sm_mhz:.0f} MHz ({peaks_kind} sm_max_mhz)",
        "algorithmic_ops_per_launch": ops_per_step * args.steps // max(1, kernel_n),
        "kernel": {1: "direct", 2: "skew", 3: "slide", 4: "column", 5: "planes"}.get(family, str(family)),
        "kernel_ms": round(kernel_ms, 4),
        "kernel_timing": "per-launch CUDA events on the launch stream, a second K-step pass "
                         f"(its steps {sum(hook_step_ms) / args.steps:.4f} ms with the events; "
                         "`value` and step_share use the event-free pass)",
        "kernel_launches": kernel_n,
        "step_share": {"kernel": round(kernel_total_ms / step_total_ms, 4),
                       "pre_pass_and_border": round(pre_ms / step_total_ms, 4),
                       "border_alone": round(border_ms / step_total_ms, 4)},
        "frac_of_step": round(ops_per_step * args.steps / (step_total_ms / 1e3) / peak_ops, 4),
        "hbm": {"achieved_gbs": round(alg_bytes * args.steps / (step_total_ms / 1e3) / 1e9, 1),
                "peak_gbs": hbm_gbs,
                "frac": round(alg_bytes * args.steps / (step_total_ms / 1e3) / 1e9 / hbm_gbs, 4),
                "bytes_per_launch": alg_bytes, "peak_kind": peaks_kind},
    }
    if executed is not None:
        roofline["executed_counts"] = executed
    if world > 1:
        roofline["note"] = "rank 0's kernel and band; job value is max over ranks"

    # ---- per-rank report (device, share, device time) ----
    mine = {"rank": rank, "device": local, **share, "ms_per_step": round(my_total_ms / args.steps, 4),
            "kernel_ms": round(kernel_ms, 4)}
    if world > 1:
        everyone = [None] * world
        dist.all_gather_object(everyone, mine)
    else:
        everyone = [mine]

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "MP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": workload_config(cfg, world),
        "roofline": roofline,
        "e2e": {"value": round(e2e_value, 2), "unit": "MP/s",
                "h2d_bytes_per_step": int(host_in.numel()) * world,
                "d2h_bytes_per_step": int(host_out.numel()) * world,
                "path": "opc_filter_rgb8_band / _batch (host pointers, pinned), "
                        f"{args.e2e_steps} steps, wall clock, max over ranks",
                "step_ms": e2e_step_ms,  # rank 0's calls one by one (a busy host shows as spread)
                "pageable": {"value": round(e2e_pageable, 2), "unit": "MP/s",
                             "path": "the same call from pageable numpy buffers (staged through "
                                     "the library's pinned ring)"}},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "ranks": everyone,
        "backend": backend if world > 1 else None,
    }
    if rank == 0 and not args.no_cpu:
        threads = host_threads()
        # rank 0's input: its band (rows [0, hi) of the image) or its first frame
        src = host_in.numpy() if F == 1 else host_in[0].numpy()
        eng = CpuEngine()
        sample = CpuSample(eng, cfg, threads, args.cpu_seconds, src=src)
        dt = sample.run()
        line["cpu_baseline"] = {"value": round(sample.megapixels / dt, 4), "unit": "MP/s",
                                "cores": threads, "kind": eng.kind,
                                "sample": sample.describe(dt)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
