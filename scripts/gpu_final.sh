# full evidence run: smoke, GPU suite, every config (+ reference arm), launch list, ncu captures
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> gpurun_out/host.txt
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
: > gpurun_out/configs.log
for c in toy hmm wsj_biphone large sweep; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-extra-e2e > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?" >> gpurun_out/configs.log
  timeout 600 python bench.py --config $c --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$c.log 2>&1; echo "$c ref rc=$?" >> gpurun_out/configs.log
done
timeout 900 python bench.py --config sweep --batch 128 --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep128.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_split_kernel" -s 2 -c 1 -o gpurun_out/prof_den python bench.py --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_den.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_linear_split" -s 2 -c 1 -o gpurun_out/prof_num python bench.py --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_num.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_streamsplit" -s 1 -c 1 -o gpurun_out/prof_ss python bench.py --config wsj_biphone --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ss.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_split_kernel" -s 2 -c 1 -o gpurun_out/prof_hmm python bench.py --config hmm --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_hmm.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
