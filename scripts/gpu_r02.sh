mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "ssplit" > gpurun_out/t_ss.log 2>&1; echo "rc=$?" >> gpurun_out/t_ss.log
timeout 900 python bench.py --config wsj_biphone --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_bi.log 2>&1
