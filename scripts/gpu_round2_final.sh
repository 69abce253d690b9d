# Full GPU test suite, then the bench lines of cfg5 (default) and cfg1-4.
cd $GRAFT_REPO_ROOT
bash scripts/gpu_tests.sh
timeout 600 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
done
for c in 1 2 3 4 5; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_cfg$c.json')); e=d['e2e']
print('cfg$c', round(d['value'],2), 'e2e', round(e['value'],2), e['ms_per_step'], e['d2h_bytes_per_step'], d['parity']['match'], d['cpu_baseline']['labels_equal_gpu'] if d.get('cpu_baseline') else None, d['clocks']['reasons'])"; done
