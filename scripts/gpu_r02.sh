# round-2: K=16 split numerators, fp64 leg, sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linear_kernel.py -q -x -p no:cacheprovider > gpurun_out/t_linear.log 2>&1; echo "rc=$?" >> gpurun_out/t_linear.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --config sweep --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep.log 2>&1
timeout 900 python bench.py --config sweep --batch 128 --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep128.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sweep128.csv python bench.py --config sweep --batch 128 --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 1800 python -m pytest tests/test_sanitizers.py -q -p no:cacheprovider -k "split or numtile" > gpurun_out/t_san.log 2>&1; echo "rc=$?" >> gpurun_out/t_san.log
