# quick iteration: planes parity tests + forced-family timing on c1/c2/c5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "planes or PLANES or forced_family or golden or fixture or criterion2 or tie or unaligned" > gpurun_out/pytest_planes.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_planes.log
rm -f gpurun_out/planes_timing.log
for k in 4 5 2; do for c in c1 c2 c5; do echo -n "k=$k " >> gpurun_out/planes_timing.log; timeout 300 python scripts/prof_run.py --config $c --kernel $k --steps 6 --frames 8 2>&1 | tail -1 >> gpurun_out/planes_timing.log; done; done
