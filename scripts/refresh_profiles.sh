#!/bin/bash
# Copy the latest profile run (scripts/gpu_profiles.sh) into profiles/ under round prefix $1 (r02).
set -e
cd "$(dirname "$0")/.."
R=${1:-r02}
cp gpurun_out/launches.csv profiles/${R}_c4_bench_launches.csv
cp gpurun_out/timing.log profiles/${R}_configs_timing.log
# algorithmic bytes per launch: filter kernels 3 B in + 3 B out per pixel; the
# shear / transpose pre-passes 3 B in + 4 B out per pixel
C4PX=$((16384*16384)); C3PX=$((4096*4096)); C5PX=$((3840*2160*64)); C2PX=$((1920*1080))
python scripts/ncu_summary.py gpurun_out/prof_c4.ncu-rep profiles/${R}_c4_skew_ncu skew $((C4PX*6)) > /dev/null
python scripts/ncu_summary.py gpurun_out/prof_c4.ncu-rep profiles/${R}_c4_shear_ncu shear $((C4PX*7)) > /dev/null
python scripts/ncu_summary.py gpurun_out/prof_c3.ncu-rep profiles/${R}_c3_slide_ncu slide_kernel $((C3PX*6)) > /dev/null
python scripts/ncu_summary.py gpurun_out/prof_c3.ncu-rep profiles/${R}_c3_transpose_ncu transpose $((C3PX*7)) > /dev/null
python scripts/ncu_summary.py gpurun_out/prof_c5.ncu-rep profiles/${R}_c5_skew_ncu skew $((C5PX*6)) > /dev/null
python scripts/ncu_summary.py gpurun_out/prof_c2.ncu-rep profiles/${R}_c2_planes_ncu planes $((C2PX*6)) > /dev/null
for c in c1 c2 c3 c4 c5; do [ -s gpurun_out/bench_$c.json ] && cp gpurun_out/bench_$c.json profiles/${R}_bench_$c.json; done
for c in c1 c2 c3 c4 c5; do [ -s gpurun_out/bench_ref_$c.json ] && cp gpurun_out/bench_ref_$c.json profiles/${R}_bench_reference_$c.json; done
R=$R python - <<'PY'
import json, os
R = os.environ["R"]
for cfg, src in (("c2", "c2_planes_ncu"), ("c3", "c3_slide_ncu"), ("c4", "c4_skew_ncu"), ("c5", "c5_skew_ncu")):
    d = json.load(open(f'profiles/{R}_{src}.json'))
    json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": d["dram_bytes_per_launch"],
               "traffic_ratio": d.get("traffic_ratio"),
               "source": f"profiles/{R}_{src}.json (ncu --set full, scripts/prof_run.py --config {cfg})"},
              open(f'profiles/{cfg}_dram_bytes.json', 'w'), indent=1)
PY
