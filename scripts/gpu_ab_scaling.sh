# band_scaling with each exp/*.so (per-share device times at N = 1, 2, 4, 8) + skew parity of each variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_scaling.log
for so in exp/*.so; do echo "== $so" >> gpurun_out/ab_scaling.log; OILPAINT_B200_LIB=$PWD/$so timeout 900 python -m pytest tests -m gpu -q -x -k "${TESTK:-skew or band or c4 or config_output}" 2>&1 | tail -1 >> gpurun_out/ab_scaling.log; done
for round in 1 2; do for so in exp/*.so; do for c in ${CFGS:-c4 c5}; do
  echo "== $so r$round" >> gpurun_out/ab_scaling.log
  OILPAINT_B200_LIB=$PWD/$so timeout 600 python scripts/band_scaling.py --config $c 1 2 4 8 >> gpurun_out/ab_scaling.log 2>&1
done; done; done
