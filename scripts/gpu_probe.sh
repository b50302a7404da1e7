# timing-only probes (exp/*.so, wrong output allowed): per-kernel event times, 2 rounds, no parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/probe.log
for round in 1 2; do for so in exp/*.so; do for c in ${CFGS:-c4}; do
  echo -n "$(basename $so) r$round $c " >> gpurun_out/probe.log
  OILPAINT_B200_LIB=$PWD/$so timeout 300 python scripts/prof_run.py --config $c --steps 6 --frames 8 --kt 2>&1 | grep -E "skew:|slide:|planes:|prepass:" | tr '\n' ' ' >> gpurun_out/probe.log
  echo >> gpurun_out/probe.log
done; done; done
