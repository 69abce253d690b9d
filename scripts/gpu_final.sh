# The round's measurement set, written under gpurun_out/ (copied to profiles/ afterwards).
cd $GRAFT_REPO_ROOT
T=${TAG:-r02}
lscpu > gpurun_out/gpu_box_host_$T.txt 2>&1; free -g >> gpurun_out/gpu_box_host_$T.txt; nvidia-smi >> gpurun_out/gpu_box_host_$T.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg5_$T.json 2> gpurun_out/bench_cfg5_$T.err
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_cfg${c}_$T.json 2>> gpurun_out/bench_cfg5_$T.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_cfg5_$T.json 2> gpurun_out/bench_reference_$T.err
timeout 900 python scripts/configs_table.py $T > gpurun_out/configs_$T.log 2>&1
timeout 900 python scripts/nd_quick.py 0 11 --time > gpurun_out/nd_engine_$T.txt 2>&1
timeout 600 python scripts/slab_scaling.py > gpurun_out/slab_scaling_$T.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg5_$T.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_$T.log 2>&1
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cull12|eval12|eval16" -c 2 -f -o gpurun_out/ball12_cfg5_$T python scripts/ab_time.py 5 > gpurun_out/ncu_full_$T.log 2>&1
echo done
