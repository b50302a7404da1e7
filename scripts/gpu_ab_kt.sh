# interleaved A/B of exp/*.so: per-kernel event times (prof_run --kt), 3 rounds; parity of each variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_kt.log
for so in exp/*.so; do echo "== $so" >> gpurun_out/ab_kt.log; OILPAINT_B200_LIB=$PWD/$so timeout 900 python -m pytest tests -m gpu -q -x -k "${TESTK:-skew or config_output}" 2>&1 | tail -1 >> gpurun_out/ab_kt.log; done
for round in 1 2 3; do for so in exp/*.so; do for c in ${CFGS:-c4}; do
  echo "$(basename $so) r$round $c" >> gpurun_out/ab_kt.log
  OILPAINT_B200_LIB=$PWD/$so timeout 300 python scripts/prof_run.py --config $c --steps 10 --frames 8 --kt 2>&1 | tail -4 >> gpurun_out/ab_kt.log
done; done; done
