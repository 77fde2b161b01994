mkdir -p gpurun_out
for np in 0 136 142 146 148; do
LFMMI_OPTIONS=tile_persist=$np timeout 900 python bench.py --config sweep --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep_np$np.log 2>&1
done
LFMMI_OPTIONS=tile_persist=142 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sweep142.csv python bench.py --config sweep --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
