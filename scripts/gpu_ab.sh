cd $GRAFT_REPO_ROOT
[ -n "$NQ" ] && timeout 600 python scripts/exact_quick.py ${NQ:-40} 7 > gpurun_out/exact_quick.log 2>&1; tail -1 gpurun_out/exact_quick.log
grep BAD gpurun_out/exact_quick.log | head -5
bash scripts/ab_run.sh 2>&1 | tee gpurun_out/ab.log | sort -k2,2 -k1,1 | awk '{print $1,$2,$5,$7,$9}'
