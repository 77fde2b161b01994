# stream split kernel: parity first, then benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "stream or large or biphone or ring" > gpurun_out/t_stream.log 2>&1; echo "rc=$?" >> gpurun_out/t_stream.log
timeout 900 python -m pytest tests/test_full_size_parity.py -q -p no:cacheprovider -k "biphone or large" > gpurun_out/t_full.log 2>&1; echo "rc=$?" >> gpurun_out/t_full.log
timeout 900 python -m pytest tests/test_sanitizers.py -q -p no:cacheprovider -k "ssplit" > gpurun_out/t_san.log 2>&1; echo "rc=$?" >> gpurun_out/t_san.log
timeout 900 python bench.py --config wsj_biphone --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_biphone.log 2>&1
LFMMI_OPTIONS=stream_mode=1024x1 timeout 900 python bench.py --config wsj_biphone --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_biphone_old.log 2>&1
timeout 900 python bench.py --config large --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_large.log 2>&1
LFMMI_OPTIONS=stream_mode=1024x2 timeout 900 python bench.py --config large --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_large_old.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fb_streamsplit_kernel" -s 1 -c 1 -o gpurun_out/prof_ssplit python bench.py --config wsj_biphone --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ss.log 2>&1
