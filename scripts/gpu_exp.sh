# usage: bash scripts/gpu_exp.sh <config> -- times every exp/*.so variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/exp.log
for so in exp/*.so; do
  echo "== $so" >> gpurun_out/exp.log
  OILPAINT_B200_LIB=$PWD/$so timeout 300 python scripts/prof_run.py --config ${1:-c4} --steps 4 >> gpurun_out/exp.log 2>&1
done
