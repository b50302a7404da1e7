# C3-only refresh of the committed evidence: GPU suite, bench lines (C3, default C4), ncu capture of the slide family, band scaling, trace
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python scripts/prof_run.py --config c3 --steps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slide_kernel|transpose|plan" -c 3 -o gpurun_out/prof_c3 -f python scripts/prof_run.py --config c3 --steps 1 > gpurun_out/ncu_c3.log 2>&1
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python scripts/band_scaling.py --config c3 1 2 4 8 > gpurun_out/band_scaling_c3.log 2>&1
if [ -f exp/trace.so ]; then OILPAINT_B200_LIB=$PWD/exp/trace.so timeout 120 python scripts/slide_trace.py > gpurun_out/slide_trace_head.log 2>&1; fi
timeout 400 python scripts/fuzz_parity.py --seconds 60 --seed 64 > gpurun_out/fuzz_head.log 2>&1
echo done > gpurun_out/refresh_c3.done
