# A/B of library builds under abl/*.so (interleaved): ball-phase median per config
cd $GRAFT_REPO_ROOT
CFGS=${CFGS:-"2 3 4 5"}
for rep in 1 2; do
for lib in abl/*.so; do
  VX_LIB_PATH=$lib REPS=${REPS:-9} timeout 600 python scripts/ab_time.py $CFGS
done
done
