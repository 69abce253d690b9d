# ad-hoc GPU call: exactness + interleaved A/B timing of the builds under abl/ (+ list statistics)
cd $GRAFT_REPO_ROOT
NQ=${NQ:-12}
for lib in abl/*.so; do
  VX_LIB_PATH=$lib timeout 600 python scripts/exact_quick.py $NQ 7 > gpurun_out/eq_$(basename $lib).log 2>&1; echo "$lib $(tail -1 gpurun_out/eq_$(basename $lib).log)"
done
CFGS="${CFGS:-2 3 5}" REPS=${REPS:-9} bash scripts/ab_run.sh 2>&1 | sort -k2,2 -k1,1 | awk '{print $1,$2,$5,$7,$9,$11}'
for lib in ${STATS_LIBS}; do VX_STATS=1 VX_LIB_PATH=$lib timeout 300 python scripts/stats_probe.py 2>&1 | head -12; done
