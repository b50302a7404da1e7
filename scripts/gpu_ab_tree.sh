# usage: bash scripts/gpu_ab_tree.sh TREE [configs...] -- interleaved timing of the in-tree library
# against an older checkout copied to TREE (exp/<name>: its package + scripts), 3 rounds
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TREE=$1; shift
CFGS=${@:-c4}
rm -f gpurun_out/ab_tree.log
for round in 1 2 3; do
  for c in $CFGS; do
    echo -n "head $c r$round " >> gpurun_out/ab_tree.log
    timeout 300 python scripts/prof_run.py --config $c --steps 6 --frames 8 2>&1 | tail -1 >> gpurun_out/ab_tree.log
    echo -n "$(basename $TREE) $c r$round " >> gpurun_out/ab_tree.log
    (cd $TREE && timeout 300 python scripts/prof_run.py --config $c --steps 6 --frames 8 2>&1 | tail -1) >> gpurun_out/ab_tree.log
  done
done
