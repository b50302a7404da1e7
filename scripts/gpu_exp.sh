# usage: bash scripts/gpu_exp.sh [configs...] -- parity subset + timing for every exp/*.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/exp.log
CFGS=${@:-c4}
for so in exp/*.so; do
  echo "== $so" >> gpurun_out/exp.log
  OILPAINT_B200_LIB=$PWD/$so timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "fixture or skew or golden or bands or criterion2" 2>&1 | tail -2 >> gpurun_out/exp.log
  for c in $CFGS; do
    OILPAINT_B200_LIB=$PWD/$so timeout 300 python scripts/prof_run.py --config $c --steps 4 --frames 8 >> gpurun_out/exp.log 2>&1
  done
done
