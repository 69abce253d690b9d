# ncu --set full of the two ball-phase kernels at cfg2, cfg3, cfg4 (one launch each)
cd $GRAFT_REPO_ROOT
T=${TAG:-r02}
for c in 2 3 4; do
  REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cull12|eval12|eval16" -c 2 -f -o gpurun_out/ball12_cfg${c}_$T python scripts/ab_time.py $c > gpurun_out/ncu_full_cfg${c}_$T.log 2>&1
  tail -1 gpurun_out/ncu_full_cfg${c}_$T.log
done
