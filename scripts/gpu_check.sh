cd $GRAFT_REPO_ROOT
bash scripts/gpu_tests.sh
timeout 900 python scripts/nd_quick.py 64 11 --time > gpurun_out/nd_quick.log 2>&1; grep -E "^bad|Gvox" gpurun_out/nd_quick.log
CFGS="2 3 4 5" REPS=7 bash scripts/ab_run.sh 2>&1 | sort -k2,2 -k1,1 | awk '{print $1,$2,$5,$7,$9}'
