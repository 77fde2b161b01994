# round-2: split numerator kernel + serial numerators for filled den batches
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv >> gpurun_out/host.txt 2>&1
timeout 900 python -m pytest tests/test_linear_kernel.py -q -x -p no:cacheprovider > gpurun_out/t_linear.log 2>&1; echo "rc=$?" >> gpurun_out/t_linear.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
B="python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline"
LFMMI_OPTIONS=linear_split=0 timeout 600 $B > gpurun_out/bench_nosplitnum.log 2>&1
timeout 900 python bench.py --config sweep --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep.log 2>&1
LFMMI_OPTIONS=serial=0 timeout 900 python bench.py --config sweep --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep_conc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_linear_split" -s 2 -c 1 -o gpurun_out/prof_num python bench.py --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_num.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
