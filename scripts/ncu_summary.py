#!/usr/bin/env python3
"""Summarise an ncu report (--set full) of the skew kernel into profiles/.

usage: python scripts/ncu_summary.py <report.ncu-rep> <out-prefix> [kernel-regex] [alg-bytes]
writes <out-prefix>.md (human summary) and <out-prefix>.json (numbers, incl.
dram bytes per launch that bench.py reports as roofline.traffic).  alg-bytes =
the kernel's algorithmic bytes per launch (input + output it must move); the
summary then states the traffic ratio dram bytes / algorithmic bytes.
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "launch__registers_per_thread": "registers",
    "launch__block_size": "block_size",
    "launch__grid_size": "grid_size",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1_data_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "l1_data_pipe_shared_pct",
    "sm__cycles_active.avg": "sm_cycles_active_avg",
    "sm__cycles_active.max": "sm_cycles_active_max",
    "sm__cycles_elapsed.avg": "sm_cycles_elapsed_avg",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def main() -> None:
    rep, prefix = sys.argv[1], sys.argv[2]
    kre = re.compile(sys.argv[3] if len(sys.argv) > 3 else "skew")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if not kre.search(name):
            continue
        d = {"kernel": name}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[key] = v * SCALE.get(units[i], 1)
        stalls = {}
        for i, h in enumerate(hdr):
            mm = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
            if mm:
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls[mm.group(1)] = round(v, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
        out.append(d)
    if not out:
        sys.exit("no matching kernel in report")
    d = out[0]
    d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
    if len(sys.argv) > 4:
        d["algorithmic_bytes_per_launch"] = float(sys.argv[4])
        d["traffic_ratio"] = round(d["dram_bytes_per_launch"] / float(sys.argv[4]), 3)
    with open(prefix + ".json", "w") as f:
        json.dump(d, f, indent=1)
    lines = [f"# ncu summary: `{d['kernel'][:80]}`", "", f"source report: `{rep}`", ""]
    if "traffic_ratio" in d:
        lines += [f"traffic ratio: {d['traffic_ratio']} (DRAM {d['dram_bytes_per_launch']:.4g} B / "
                  f"algorithmic {d['algorithmic_bytes_per_launch']:.4g} B per launch)", ""]
    lines += ["| metric | value |", "|---|---|"]
    for k, v in d.items():
        if k in ("kernel", "stalls_per_issue"):
            continue
        lines.append(f"| {k} | {v:.6g} |" if isinstance(v, float) else f"| {k} | {v} |")
    lines += ["", "stall reasons (warps stalled per issued instruction):", ""]
    lines += [f"- {k}: {v}" for k, v in d["stalls_per_issue"].items()]
    with open(prefix + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
