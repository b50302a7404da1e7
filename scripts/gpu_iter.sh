# usage: bash scripts/gpu_iter.sh [ncu]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/timing.log
for c in c1 c2 c3 c4; do timeout 300 python scripts/prof_run.py --config $c --steps 3 >> gpurun_out/timing.log 2>&1; done
timeout 300 python scripts/prof_run.py --config c5 --steps 3 --frames 8 >> gpurun_out/timing.log 2>&1
if [ "$1" = "ncu" ]; then
timeout 300 python scripts/prof_run.py --config c4 --steps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skew -c 1 -o gpurun_out/prof_skew_c4 -f python scripts/prof_run.py --config c4 --steps 1 > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
fi
if [ "$1" = "launches" ]; then
timeout 300 python scripts/prof_run.py --config c4 --steps 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_run.py --config c4 --steps 2 > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
fi
