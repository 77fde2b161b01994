mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "configs or c2 or golden" > gpurun_out/pytest_den.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_den.log
for i in 1 2 3; do timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_den_$i.log 2>&1; done
