# usage: bash scripts/gpu_prof_exp.sh [config] [frames] -- one ncu --set full capture of the skew kernel per exp/*.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${1:-c4}
FR=${2:-0}
for so in exp/*.so; do
  n=$(basename $so .so)
  OILPAINT_B200_LIB=$PWD/$so timeout 300 python scripts/prof_run.py --config $CFG --steps 1 --frames $FR > gpurun_out/plain_$n.log 2>&1 && \
  OILPAINT_B200_LIB=$PWD/$so timeout 900 ncu --set full --clock-control none --import-source on -k regex:skew -c 1 -o gpurun_out/prof_${n}_$CFG -f python scripts/prof_run.py --config $CFG --steps 1 --frames $FR > gpurun_out/ncu_$n.log 2>&1
  echo "$n ncu rc=$?" >> gpurun_out/ncu_exp.log
done
