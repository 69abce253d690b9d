cd $GRAFT_REPO_ROOT
timeout 900 python scripts/nd_quick.py ${NQ:-64} 11 --time > gpurun_out/nd_quick.log 2>&1
grep -E "BAD|bad|Gvox|Error|error" gpurun_out/nd_quick.log | head -30
