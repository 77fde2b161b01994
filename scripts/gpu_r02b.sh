# new GPU tests + N = 2 bench plumbing on one GPU (gloo) + large-config stream modes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "ragged_steps or all_failed or bad_lengths" > gpurun_out/t_new.log 2>&1; echo "rc=$?" >> gpurun_out/t_new.log
BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config sweep --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_sweep.log
BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_wsj.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_wsj.log
BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --impl reference --steps 1 --warmup 1 > gpurun_out/bench_n2_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_ref.log
L="python bench.py --config large --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline"
for m in 1024x1 512x2 split; do LFMMI_OPTIONS=stream_mode=$m timeout 900 $L > gpurun_out/large_$m.log 2>&1; done
