cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_run.py --config c3 --steps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slide" -c 1 -o gpurun_out/prof_c3 -f python scripts/prof_run.py --config c3 --steps 1 > gpurun_out/ncu_c3.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3.log
