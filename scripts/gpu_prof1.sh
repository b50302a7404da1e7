cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c1 c2 c3 c4; do timeout 300 python scripts/prof_run.py --config $c --steps 3 >> gpurun_out/timing.log 2>&1; done
timeout 300 python scripts/prof_run.py --config c5 --steps 3 --frames 8 >> gpurun_out/timing.log 2>&1
timeout 300 python scripts/prof_run.py --config c4 --steps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skew -c 1 -o gpurun_out/prof_skew_c4 python scripts/prof_run.py --config c4 --steps 1 > gpurun_out/ncu.log 2>&1
echo "done rc=$?" >> gpurun_out/ncu.log
