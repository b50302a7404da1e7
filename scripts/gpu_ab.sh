# usage: bash scripts/gpu_ab.sh [configs...] -- interleaved A/B timing of exp/*.so (3 rounds), no tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
CFGS=${@:-c4}
for round in 1 2 3; do
  for so in exp/*.so; do
    for c in $CFGS; do
      echo -n "$(basename $so) r$round " >> gpurun_out/ab.log
      OILPAINT_B200_LIB=$PWD/$so timeout 300 python scripts/prof_run.py --config $c --steps 6 --frames 8 2>&1 | tail -1 >> gpurun_out/ab.log
    done
  done
done
