mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_linear_kernel.py tests/test_gpu_parity.py tests/test_full_size_parity.py -q -p no:cacheprovider -x -k "biphone or large or linear or l2_path or stream" > gpurun_out/t_emit.log 2>&1; echo "rc=$?" >> gpurun_out/t_emit.log
timeout 600 python bench.py --config wsj_biphone --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_bi.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_mono.log 2>&1
