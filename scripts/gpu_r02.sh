mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linear_kernel.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "linear or configs or packed" > gpurun_out/t_linear.log 2>&1; echo "rc=$?" >> gpurun_out/t_linear.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
S="python bench.py --config sweep --batch 128 --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline"
for nc in 64 66 68; do LFMMI_OPTIONS=split_clusters=$nc timeout 600 $S > gpurun_out/sw128_nc$nc.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sw128.csv python bench.py --config sweep --batch 128 --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch2.log 2>&1
