cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/pageable_ab.log
for round in 1 2; do for so in exp/*.so; do
  echo "== $so" >> gpurun_out/pageable_ab.log
  OILPAINT_B200_LIB=$PWD/$so timeout 600 python scripts/pageable_probe.py >> gpurun_out/pageable_ab.log 2>&1
done; done
