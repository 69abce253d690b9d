cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1_ref.json 2> gpurun_out/r1_ref.err
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/r1_bench_c$c.json 2>> gpurun_out/r1_bench.err; done
