mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_linear_kernel.py -q -p no:cacheprovider -x > gpurun_out/t_lin.log 2>&1; echo "rc=$?" >> gpurun_out/t_lin.log
timeout 1200 python -m pytest tests/test_sanitizers.py -q -p no:cacheprovider -k "lin16" > gpurun_out/t_san.log 2>&1; echo "rc=$?" >> gpurun_out/t_san.log
timeout 900 python bench.py --config sweep --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep.log 2>&1
LFMMI_OPTIONS=linear_k16w=1 timeout 900 python bench.py --config sweep --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep_w1.log 2>&1
timeout 600 python bench.py --config sweep --batch 128 --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep128.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sweep.csv python bench.py --config sweep --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
