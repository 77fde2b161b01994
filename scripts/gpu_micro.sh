mkdir -p gpurun_out
./scripts/micro/post_scatter > gpurun_out/micro_post_scatter.log 2>&1
B="python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/bench_nc71.log 2>&1
timeout 900 python bench.py --config sweep --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep.log 2>&1
LFMMI_OPTIONS=split=1 timeout 900 python bench.py --config sweep --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep_split.log 2>&1
