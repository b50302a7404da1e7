# ncu captures for profiles/: skew + shear (C4), slide + transpose (C3), skew (C5, 64 frames),
# planes (C2), launch list (bench C4), clocked bench lines for C1-C5 and the reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/timing.log
for c in c1 c2 c3 c4; do timeout 300 python scripts/prof_run.py --config $c --steps 6 >> gpurun_out/timing.log 2>&1; done
timeout 300 python scripts/prof_run.py --config c5 --steps 3 >> gpurun_out/timing.log 2>&1
timeout 300 python scripts/prof_run.py --config c4 --steps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skew|shear" -c 2 -o gpurun_out/prof_c4 -f python scripts/prof_run.py --config c4 --steps 1 > gpurun_out/ncu_c4.log 2>&1
timeout 300 python scripts/prof_run.py --config c3 --steps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slide_kernel|transpose|plan" -c 3 -o gpurun_out/prof_c3 -f python scripts/prof_run.py --config c3 --steps 1 > gpurun_out/ncu_c3.log 2>&1
timeout 300 python scripts/prof_run.py --config c5 --steps 1 > gpurun_out/plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skew" -c 1 -o gpurun_out/prof_c5 -f python scripts/prof_run.py --config c5 --steps 1 > gpurun_out/ncu_c5.log 2>&1
timeout 300 python scripts/prof_run.py --config c2 --steps 1 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"planes" -c 1 -o gpurun_out/prof_c2 -f python scripts/prof_run.py --config c2 --steps 1 > gpurun_out/ncu_c2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/plain_b.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
for c in c1 c2 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in c1 c2 c3 c4 c5; do timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/bench_ref_$c.json 2> gpurun_out/bench_ref_$c.err; done
echo done > gpurun_out/profiles.done
