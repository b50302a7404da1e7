# planes parity tests (in-tree lib + every exp/*.so) + A/B timing (L2 flushed) of exp/*.so with the planes family forced
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/pytest_planes.log gpurun_out/ab_planes.log
SEL="planes or PLANES or forced_family or golden or fixture or criterion2 or tie or unaligned"
timeout 900 python -m pytest tests -m gpu -q -x -k "$SEL" 2>&1 | tail -2 >> gpurun_out/pytest_planes.log
for so in exp/*.so; do echo "== $so" >> gpurun_out/pytest_planes.log; OILPAINT_B200_LIB=$PWD/$so timeout 900 python -m pytest tests -m gpu -q -x -k "planes or PLANES or forced_family" 2>&1 | tail -2 >> gpurun_out/pytest_planes.log; done
for c in ${CFGS:-c2 c1}; do timeout 900 python scripts/ab_time.py --config $c --kernel ${KERNEL:-5} --rounds 3 --frames 8 exp/*.so >> gpurun_out/ab_planes.log 2>&1; done
