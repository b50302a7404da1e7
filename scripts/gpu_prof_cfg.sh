# usage: bash scripts/gpu_prof_cfg.sh <config> <frames> <kernel-regex> -- one ncu --set full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_run.py --config $1 --steps 1 --frames $2 > gpurun_out/plain_$1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$3" -c 1 -o gpurun_out/prof_$1 -f python scripts/prof_run.py --config $1 --steps 1 --frames $2 > gpurun_out/ncu_$1.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$1.log
