mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_kernel_seam.py -q -x -p no:cacheprovider > gpurun_out/pytest_den.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_den.log
for i in 1 2; do LFMMI_DEBUG=1 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_den_$i.log 2>&1; done
timeout 900 python scripts/time_passes.py sweep > gpurun_out/passes.log 2>&1
