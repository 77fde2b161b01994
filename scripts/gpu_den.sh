mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "configs or c2 or golden or three_phase or packed" > gpurun_out/pytest_den.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_den.log
for i in 1 2; do LFMMI_DEBUG=1 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_den_$i.log 2>&1; done
LFMMI_TILE_SINGLE_X=1 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_den_1x.log 2>&1
