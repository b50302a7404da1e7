# ncu --set full of the planes kernel on c2 (and c5, 8 frames with PL5=1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"planes" -c 1 -o gpurun_out/prof_planes_c2 -f python scripts/prof_run.py --config c2 --kernel 5 --steps 1 > gpurun_out/ncu_pl2.log 2>&1
[ -n "$PL5" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"planes" -c 1 -o gpurun_out/prof_planes_c5 -f python scripts/prof_run.py --config c5 --kernel 5 --steps 1 --frames 8 > gpurun_out/ncu_pl5.log 2>&1
exit 0
