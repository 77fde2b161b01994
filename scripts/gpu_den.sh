mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "configs or c2 or golden or three_phase" > gpurun_out/pytest_den.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_den.log
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_den_$i.log 2>&1; done
