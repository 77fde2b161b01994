# round-2 iteration: new-kernel tests first (fast feedback), bench (default + A/B
# variants), full GPU suite, ncu launch list + capture of the numerator kernel
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv >> gpurun_out/host.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_linear_kernel.py -q -x -p no:cacheprovider > gpurun_out/t_linear.log 2>&1; echo "rc=$?" >> gpurun_out/t_linear.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "stream or large" > gpurun_out/t_stream.log 2>&1; echo "rc=$?" >> gpurun_out/t_stream.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
LFMMI_LIB_VARIANT=rows8 timeout 600 python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_rows8.log 2>&1; echo "rc=$?" >> gpurun_out/bench_rows8.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_again.log 2>&1; echo "rc=$?" >> gpurun_out/bench_again.log
timeout 900 python bench.py --config wsj_biphone --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_biphone.log 2>&1; echo "rc=$?" >> gpurun_out/bench_biphone.log
LFMMI_OPTIONS=stream_ring=0 timeout 900 python bench.py --config wsj_biphone --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_biphone_noring.log 2>&1; echo "rc=$?" >> gpurun_out/bench_biphone_noring.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_linear_kernel" -s 2 -c 1 -o gpurun_out/prof_num python bench.py --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_num.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
