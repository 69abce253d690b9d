cd $GRAFT_REPO_ROOT
for lib in abl/*.so; do
  VX_LIB_PATH=$lib timeout 600 python scripts/exact_quick.py ${NQ:-20} 7 > gpurun_out/eq_$(basename $lib).log 2>&1; echo "$lib $(tail -1 gpurun_out/eq_$(basename $lib).log)"
done
bash scripts/ab_run.sh 2>&1 | sort -k2,2 -k1,1 | awk '{print $1,$2,$5,$7,$9,$11}'
