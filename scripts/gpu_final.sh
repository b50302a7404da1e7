# end-of-round refresh: GPU suite, smoke, ncu captures, launch list, bench lines
# and reference arm for all five configs, per-config band scaling, the
# reference acceptance suite and sweep with EngineKind::Cuda
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash scripts/gpu_profiles.sh
rm -f gpurun_out/band_scaling.log
for c in c1 c2 c3 c4 c5; do timeout 600 python scripts/band_scaling.py --config $c 1 2 4 8 >> gpurun_out/band_scaling.log 2>&1; done
timeout 900 build/integration/ref_acceptance_cuda > gpurun_out/ref_acceptance.log 2>&1
timeout 900 build/integration/sweep_cuda --sizes vga,svga,xga,fhd,wqxga --radii 2,4,6,8 --reps 5 > gpurun_out/ref_sweep.csv 2> gpurun_out/ref_sweep.err
echo done > gpurun_out/final.done
