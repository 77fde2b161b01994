# round-2 iteration: emissions pre-pass (E shared by the linear numerator and split
# den kernels), stream ring v2; tests first, then A/B benches, ncu, full suite
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv >> gpurun_out/host.txt 2>&1
timeout 900 python -m pytest tests/test_linear_kernel.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/t_fast.log 2>&1; echo "rc=$?" >> gpurun_out/t_fast.log
B="python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline"
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
LFMMI_OPTIONS=emit=0 timeout 600 $B > gpurun_out/bench_noemit.log 2>&1
LFMMI_OPTIONS=chore_bias=8 timeout 600 $B > gpurun_out/bench_bias8.log 2>&1
LFMMI_OPTIONS=chore_bias=2 timeout 600 $B > gpurun_out/bench_bias2.log 2>&1
LFMMI_OPTIONS=split_clusters=69 timeout 600 $B > gpurun_out/bench_nc69.log 2>&1
LFMMI_OPTIONS=split_clusters=74 timeout 600 $B > gpurun_out/bench_nc74.log 2>&1
timeout 600 $B > gpurun_out/bench_again.log 2>&1
timeout 900 python bench.py --config wsj_biphone --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_biphone.log 2>&1
LFMMI_OPTIONS=stream_ring=0 timeout 900 python bench.py --config wsj_biphone --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_biphone_noring.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_split_kernel" -s 2 -c 1 -o gpurun_out/prof_den python bench.py --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_den.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_linear_kernel" -s 2 -c 1 -o gpurun_out/prof_num python bench.py --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_num.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fb_stream_kernel" -s 1 -c 1 -o gpurun_out/prof_stream_ring python bench.py --config wsj_biphone --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_stream.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
