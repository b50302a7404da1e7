"""bench.py's measurement helpers (CPU): the SURVEY.md 8(d) roofline models,
the L2-flush rule and the per-rank input bytes of a multi-GPU split."""
from __future__ import annotations

import importlib.util
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("opc_bench", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_best_fit_models_match_survey_table(bench):
    # SURVEY.md 8(d) "1-GPU roof" table: the cheapest model per config
    assert bench.best_fit_model(2, 21) == ("slide", 145)     # C1
    assert bench.best_fit_model(5, 21) == ("slide", 229)     # C2
    assert bench.best_fit_model(10, 257) == ("slide", 1077)  # C3
    assert bench.best_fit_model(15, 21) == ("colhist", 257)  # C4
    assert bench.best_fit_model(7, 31) == ("slide", 315)     # C5
    assert bench.colhist_ops_per_px(21) == 257
    # radius 0 with very few bins: the direct scan is the cheapest model
    assert bench.best_fit_model(0, 2) == ("direct", 7 + 4 * 2 + 12)


def test_l2_rule_and_rank_bytes(bench):
    CONFIGS = bench.load_workloads()
    c4 = CONFIGS["c4"]
    assert bench.rank0_in_bytes(c4, 1) == 3 * 16384 * 16384
    # rank 0 of 8: its 2048 rows plus the 15 halo rows below
    assert bench.rank0_in_bytes(c4, 8) == (2048 + 15) * 16384 * 3
    assert bench.rank0_in_bytes(CONFIGS["c5"], 8) == 8 * 3840 * 2160 * 3
    assert "no flush" in bench.workload_config(c4, 1)["l2"]
    assert "flushed" in bench.workload_config(c4, 8)["l2"]
    assert "flushed" in bench.workload_config(CONFIGS["c1"], 1)["l2"]
    cfg = bench.workload_config(CONFIGS["c5"], 2)
    assert cfg["partition"].startswith("frames") and cfg["frames"] == 64


def test_workloads_match_package_configs(bench):
    from paper_1405_1020_b200.patterns import CONFIGS
    wl = bench.load_workloads()
    assert set(wl) == set(CONFIGS) == {"c1", "c2", "c3", "c4", "c5"}
    for k, w in wl.items():
        c = CONFIGS[k]
        assert (c.width, c.height, c.frames, c.radius, c.levels, c.pattern, c.seed) == \
            (w.width, w.height, w.frames, w.radius, w.levels, w.pattern, w.seed)


PURITY = r"""
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--config", sys.argv[1], "--steps", "1",
            "--warmup", "0", "--gpus", "2"]
runpy.run_path("bench.py", run_name="__main__")
assert not any(m == "paper_1405_1020_b200" or m.startswith("paper_1405_1020_b200.")
               for m in sys.modules), "reference arm imported the product package"
maps = open("/proc/self/maps").read()
assert "liboilpaint_b200" not in maps, "reference arm mapped the product library"
print("PURE", "libref_oilpaint" in maps)
"""


@pytest.mark.parametrize("config", ["c1", "c3"])
def test_reference_arm_never_loads_the_product(config):
    """bench.py --impl reference runs the reference engine (oracle/_ref) on
    inputs it generates itself: it imports no product module and maps no
    product library (the ratio is void otherwise)."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, OILPAINT_REF_STEP_S="0.05", OILPAINT_B200_AUTOBUILD="0")
    res = subprocess.run([sys.executable, "-c", PURITY, config], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    lines = res.stdout.strip().splitlines()
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert lines[-1].startswith("PURE")


def test_reference_inputs_match_product_generators(bench):
    """The reference arm's inputs (oracle/_ref: the reference Noise generator,
    the harness generators) are the bytes the product arm generates."""
    import numpy as np
    import paper_1405_1020_b200 as opc
    eng = bench.CpuEngine()
    if eng.ref is None:
        pytest.skip("oracle/_ref not built")
    for name in ("c1", "c2", "c3", "c4", "c5"):
        wl = bench.load_workloads()[name]
        got = eng.generate_rows(wl, 40)
        want = opc.CONFIGS[name].generate_rows(0, 40)
        assert np.array_equal(got, want), name


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c2", "c5"])
def test_bench_gpus2_relaunches_two_ranks(config):
    """`bench.py --gpus 2` run plainly (as the driver's scaling run does)
    relaunches itself as 2 ranks under torch.distributed.run.  On a 1-GPU box
    the ranks share the device over gloo (OPC_BENCH_BACKEND=gloo: a plumbing
    check, not a number): n_gpus 2, the row-band split of
    proj/src/parallel.cpp:55-108 lifted to ranks (C2) or the frame split (C5),
    and a cpu_baseline on the line."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, OPC_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", config,
                          "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--cpu-seconds", "1"],
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 prints the one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["cpu_baseline"]["value"] > 0
    ranks = sorted(d["ranks"], key=lambda x: x["rank"])
    assert [x["rank"] for x in ranks] == [0, 1]
    if config == "c2":
        assert ranks[0]["rows"] == [0, 540] and ranks[1]["rows"] == [540, 1080]
        assert ranks[0]["input_rows"] == [0, 545] and ranks[1]["input_rows"] == [535, 1080]
    else:
        assert ranks[0]["frames"] == [0, 32] and ranks[1]["frames"] == [32, 64]
