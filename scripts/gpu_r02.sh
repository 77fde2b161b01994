mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_full_size_parity.py -q -p no:cacheprovider -x > gpurun_out/t_par.log 2>&1; echo "rc=$?" >> gpurun_out/t_par.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_mono.log 2>&1
timeout 600 python bench.py --config hmm --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_hmm.log 2>&1
LFMMI_OPTIONS=split_small=0 timeout 600 python bench.py --config hmm --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_hmm16.log 2>&1
timeout 600 python bench.py --config sweep --batch 128 --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep128.log 2>&1
timeout 900 python bench.py --config sweep --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep.log 2>&1
timeout 600 python scripts/host_overhead.py hmm wsj_mono > gpurun_out/host_overhead.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hmm.csv python bench.py --config hmm --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
