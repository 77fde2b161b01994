mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_full_size_parity.py -q -p no:cacheprovider -k "hmm" > gpurun_out/t_hmm.log 2>&1; echo "rc=$?" >> gpurun_out/t_hmm.log
timeout 900 python bench.py --config hmm --steps 20 --warmup 3 --no-extra-e2e > gpurun_out/bench_hmm.log 2>&1
timeout 600 python bench.py --config hmm --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_hmm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hmm.csv python bench.py --config hmm --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
