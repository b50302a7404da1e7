# full GPU suite + device-resident timing of the planner's choice vs forced families
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
rm -f gpurun_out/ab_default.log
for c in c1 c2 c5; do for k in 0 2 4; do timeout 900 python scripts/ab_time.py --config $c --kernel $k --rounds 2 --frames 8 default >> gpurun_out/ab_default.log 2>&1; done; done
