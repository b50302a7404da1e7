cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/small.log
for c in c1 c2 c3; do for k in 1 2; do timeout 300 python scripts/prof_run.py --config $c --steps 4 --kernel $k >> gpurun_out/small.log 2>&1; done; done
timeout 300 python scripts/prof_run.py --config c5 --steps 3 --frames 8 --kernel 1 >> gpurun_out/small.log 2>&1
