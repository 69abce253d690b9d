cd $GRAFT_REPO_ROOT
CFG=${CFG:-5}
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cull12|eval12|eval16" -c 2 -f -o gpurun_out/ball12_cfg$CFG python scripts/ab_time.py $CFG > gpurun_out/ncu12.log 2>&1
tail -2 gpurun_out/ncu12.log
