# round-2 iteration: validate defaults (69 clusters, ring off), cluster sweep,
# reference arm, full suite
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv >> gpurun_out/host.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
B="python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline"
for nc in 66 68 70 71 72; do LFMMI_OPTIONS=split_clusters=$nc timeout 600 $B > gpurun_out/bench_nc$nc.log 2>&1; done
LFMMI_OPTIONS=chore_bias=8 timeout 600 $B > gpurun_out/bench_bias8.log 2>&1
timeout 600 $B > gpurun_out/bench_again.log 2>&1
timeout 900 python bench.py --config sweep --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_sweep.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
