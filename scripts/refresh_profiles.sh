#!/bin/bash
# Copy the latest full GPU run (scripts/gpu_full.sh + scripts/gpu_profiles.sh) into profiles/.
set -e
cd "$(dirname "$0")/.."
cp gpurun_out/bench.json profiles/r01_bench_c4.json
cp gpurun_out/bench_ref.json profiles/r01_bench_reference_c4.json
cp gpurun_out/launches.csv profiles/r01_c4_bench_launches.csv
cp gpurun_out/timing.log profiles/r01_configs_timing.log
for k in skew shear; do python scripts/ncu_summary.py gpurun_out/prof_c4.ncu-rep profiles/r01_c4_${k}_ncu $k > /dev/null; done
for k in slide transpose; do python scripts/ncu_summary.py gpurun_out/prof_c3.ncu-rep profiles/r01_c3_${k}_ncu $k > /dev/null; done
python scripts/ncu_summary.py gpurun_out/prof_c5.ncu-rep profiles/r01_c5_skew_ncu skew > /dev/null
python scripts/ncu_summary.py gpurun_out/prof_c2.ncu-rep profiles/r01_c2_column_ncu column > /dev/null
for c in c1 c2 c3 c5; do [ -s gpurun_out/bench_$c.json ] && cp gpurun_out/bench_$c.json profiles/r01_bench_$c.json; done
for c in c1 c2 c3 c5; do [ -s gpurun_out/bench_ref_$c.json ] && cp gpurun_out/bench_ref_$c.json profiles/r01_bench_reference_$c.json; done
python - <<'PY'
import json
d = json.load(open('profiles/r01_c4_skew_ncu.json'))
json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": d["dram_bytes_per_launch"],
           "source": "profiles/r01_c4_skew_ncu.json (ncu --set full, scripts/prof_run.py --config c4)"},
          open('profiles/c4_dram_bytes.json', 'w'), indent=1)
for cfg, src in (("c2", "r01_c2_column_ncu"), ("c3", "r01_c3_slide_ncu"), ("c5", "r01_c5_skew_ncu")):
    d = json.load(open(f'profiles/{src}.json'))
    json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": d["dram_bytes_per_launch"],
               "source": f"profiles/{src}.json (ncu --set full, scripts/prof_run.py --config {cfg})"},
              open(f'profiles/{cfg}_dram_bytes.json', 'w'), indent=1)
PY
