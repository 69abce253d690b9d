# ad-hoc GPU call: bench (clock sampler check) + ncu capture of the ball kernels at cfg5
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_cfg5_now.json 2> gpurun_out/bench_cfg5_now.err
python -c "import json;d=json.load(open('gpurun_out/bench_cfg5_now.json'));print(d['value'],d['clocks'],d['stage_ms'])"
CFG=5 bash scripts/gpu_ncu12.sh
