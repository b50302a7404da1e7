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
    from paper_1405_1020_b200.patterns import CONFIGS
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
