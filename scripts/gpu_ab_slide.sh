# A/B of exp/*.so on the slide family: parity subset (short timeout: a ring-protocol bug hangs), then C3 kernel times, 3 rounds
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_slide.log
for so in exp/*.so; do echo "== $so" >> gpurun_out/ab_slide.log; OILPAINT_B200_LIB=$PWD/$so timeout 150 python -m pytest tests -m gpu -q -x -k "${TESTK:-slide or config_output or fixture or levels_256}" 2>&1 | tail -2 >> gpurun_out/ab_slide.log; done
for round in 1 2 3; do for so in exp/*.so; do
  echo -n "$(basename $so) r$round " >> gpurun_out/ab_slide.log
  OILPAINT_B200_LIB=$PWD/$so timeout 60 python scripts/prof_run.py --config c3 --steps 10 --kt 2>&1 | grep -E "slide:" | tr '\n' ' ' >> gpurun_out/ab_slide.log
  echo >> gpurun_out/ab_slide.log
done; done
cat gpurun_out/ab_slide.log
