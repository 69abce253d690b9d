cd $GRAFT_REPO_ROOT
bash scripts/gpu_tests.sh
CFGS="1 2 5" REPS=7 bash scripts/ab_run.sh 2>&1 | sort -k2,2 -k1,1 | awk '{print $1,$2,$5,$7,$9}'
python scripts/slab_scaling.py 2>&1 | tail -4
