# every engine path on small cases with the bounds-checked debug build (VX_DEBUG asserts), then the release build
cd $GRAFT_REPO_ROOT
VX_LIB=debug timeout 1200 python scripts/sanitize_cases.py > gpurun_out/sanitize_debug.log 2>&1; echo "debug rc=$?"; tail -2 gpurun_out/sanitize_debug.log
timeout 1200 python scripts/sanitize_cases.py > gpurun_out/sanitize_release.log 2>&1; echo "release rc=$?"; tail -2 gpurun_out/sanitize_release.log
