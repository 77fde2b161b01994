mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "configs or numerator_group or packed" > gpurun_out/pytest_sweep.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sweep.log
timeout 300 python bench.py --config sweep --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sweep_room.log 2>&1
LFMMI_NO_NUM_ROOM=1 timeout 300 python bench.py --config sweep --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sweep_noroom.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_den_1.log 2>&1
