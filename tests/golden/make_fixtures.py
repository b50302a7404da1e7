#!/usr/bin/env python3
"""Regenerates the committed parity fixtures in tests/golden/ FROM THE REFERENCE.

Run in the build container (needs /root/reference and the oracle/_ref build):

  python tests/golden/make_fixtures.py golden    # gradient8_r2_l20_zero.ppm
  python tests/golden/make_fixtures.py cases     # ref_cases.npz
  python tests/golden/make_fixtures.py digests   # config_digests.json (minutes)

golden  : copies the reference's own generator proj/tests/golden/make_golden.py
          to a scratch directory (it writes next to itself), runs it there and
          copies the 203-byte PPM here.  The reference tree is never written.
cases   : random small images (criterion-1/2 style, plus L=256 and large-radius
          cases); outputs computed by the UNMODIFIED reference library in
          oracle/_ref: apply_sequential / apply_parallel, and oracle::filter
          (proj/tests/support/oracle.cpp) for L=256.
digests : SHA-256 of every BASELINE config input (our generators) and of the
          reference output for it (apply_parallel with all host threads; config
          3 through the reference's parallel_for_rows + filter_pixel body since
          validate rejects L=256), so the GPU box can check full-size outputs
          bit-exactly without the minutes-long CPU run.
"""
from __future__ import annotations

import hashlib
import json
import shutil
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib  # noqa: E402

REF_GOLDEN_SCRIPT = Path("/root/reference/proj/tests/golden/make_golden.py")


def make_golden() -> None:
    with tempfile.TemporaryDirectory() as tmp:
        script = Path(tmp) / "make_golden.py"
        shutil.copy(REF_GOLDEN_SCRIPT, script)
        subprocess.run([sys.executable, str(script)], check=True, cwd=tmp)
        ppm = Path(tmp) / "gradient8_r2_l20_zero.ppm"
        shutil.copy(ppm, HERE / "gradient8_r2_l20_zero.ppm")
    print("wrote", HERE / "gradient8_r2_l20_zero.ppm")


def make_cases() -> None:
    ref = oracle_lib.load_ref()
    rng = np.random.default_rng(20261019)
    metas, ins, outs = [], [], []

    def add(img, r, L, border, engine):
        h, w, _ = img.shape
        if L == 256:
            out = oracle_lib.ref_oracle_filter(ref, img, r, L, border)
            src = 2
        else:
            out = oracle_lib.ref_apply(ref, img, r, L, border, engine=engine,
                                       workers=4 if engine else 0)
            src = engine
        metas.append((w, h, r, L, border, src))
        ins.append(img.reshape(-1))
        outs.append(out.reshape(-1))

    # criterion 1 style (proj/tests/acceptance.cpp:44-67): w,h <= 16, r <= 3.
    for _ in range(240):
        w, h = int(rng.integers(1, 17)), int(rng.integers(1, 17))
        max_r = min(3, (min(w, h) - 1) // 2)
        r = int(rng.integers(0, max_r + 1))
        L = int(rng.choice([1, 10, 20, 255]))
        add(rng.integers(0, 256, (h, w, 3), dtype=np.uint8), r, L, int(rng.integers(0, 2)), 0)
    # criterion 2 style (acceptance.cpp:71-101): w,h <= 96, r <= 5, parallel engine.
    for _ in range(24):
        w, h = int(rng.integers(1, 97)), int(rng.integers(1, 97))
        max_r = min(5, (min(w, h) - 1) // 2)
        r = int(rng.integers(0, max_r + 1))
        L = int(rng.choice([1, 20, 30, 255]))
        add(rng.integers(0, 256, (h, w, 3), dtype=np.uint8), r, L, int(rng.integers(0, 2)), 1)
    # L = 256 (config-3 extension) through oracle::filter.
    for _ in range(16):
        w, h = int(rng.integers(3, 33)), int(rng.integers(3, 33))
        r = int(rng.integers(0, min(4, (min(w, h) - 1) // 2) + 1))
        add(rng.integers(0, 256, (h, w, 3), dtype=np.uint8), r, 256, int(rng.integers(0, 2)), 0)
    # Large radii around the 64-bit packing limit (r = 15) and beyond.
    for r in (12, 15, 16, 20):
        for L in (20, 31):
            w, h = 2 * r + 1 + int(rng.integers(0, 24)), 2 * r + 1 + int(rng.integers(0, 24))
            add(rng.integers(0, 256, (h, w, 3), dtype=np.uint8), r, L, 0, 1)
    # Smooth / flat content: many ties and single-bin windows.
    for _ in range(8):
        w, h = int(rng.integers(20, 64)), int(rng.integers(20, 64))
        base = rng.integers(0, 256, 3)
        img = np.clip(base + rng.integers(-6, 7, (h, w, 3)), 0, 255).astype(np.uint8)
        add(img, int(rng.integers(1, 6)), int(rng.choice([20, 30, 255])), 0, 0)

    meta = np.array(metas, np.int32)
    np.savez_compressed(HERE / "ref_cases.npz", meta=meta, inputs=np.concatenate(ins),
                        outputs=np.concatenate(outs))
    print("wrote", HERE / "ref_cases.npz", len(metas), "cases")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(memoryview(np.ascontiguousarray(a)).cast("B")).hexdigest()


def make_digests(names: list[str]) -> None:
    from paper_1405_1020_b200.patterns import CONFIGS

    ref = oracle_lib.load_ref()
    threads = oracle_lib.cpu_count()
    path = HERE / "config_digests.json"
    data = json.loads(path.read_text()) if path.exists() else {}
    for name in names:
        cfg = CONFIGS[name]
        entry = {"width": cfg.width, "height": cfg.height, "frames": cfg.frames,
                 "radius": cfg.radius, "levels": cfg.levels, "pattern": int(cfg.pattern),
                 "seed": cfg.seed, "inputs": [], "outputs": {}}
        borders = [0, 1] if name in ("c1", "c2") else [0]
        out_h = {b: [] for b in borders}
        t0 = time.time()
        for f in range(cfg.frames):
            img = cfg.generate(f)
            entry["inputs"].append(sha(img))
            for b in borders:
                if cfg.levels == 256:
                    out = np.empty_like(img)
                    h, w, _ = img.shape
                    rc = ref.ref_filter_rows_any_levels(img.ctypes.data, out.ctypes.data, w, h,
                                                        cfg.radius, cfg.levels, b, threads)
                    assert rc == 0, ref.ref_last_error()
                else:
                    out = oracle_lib.ref_apply(ref, img, cfg.radius, cfg.levels, b, engine=1,
                                               workers=threads)
                out_h[b].append(sha(out))
        for b in borders:
            entry["outputs"]["copy_input" if b == 0 else "zero_fill"] = out_h[b]
        entry["reference_engine"] = ("parallel_for_rows+filter_pixel (L=256)" if cfg.levels == 256
                                     else "apply_parallel")
        entry["cpu_seconds"] = round(time.time() - t0, 1)
        entry["threads"] = threads
        data[name] = entry
        path.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
        print(name, "done in", entry["cpu_seconds"], "s")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("golden", "all"):
        make_golden()
    if what in ("cases", "all"):
        make_cases()
    if what in ("digests", "all"):
        make_digests(sys.argv[2:] or ["c1", "c2", "c3", "c5", "c4"])
