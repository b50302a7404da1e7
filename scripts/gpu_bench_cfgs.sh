# clocked bench lines for the given configs (default c1 c2 c5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CFGS:-c1 c2 c5}; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
