# round-2: sanitizers after the named-barrier fix, stream ring v3 A/B, full suite
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_sanitizers.py -q -p no:cacheprovider > gpurun_out/t_san.log 2>&1; echo "rc=$?" >> gpurun_out/t_san.log
B="python bench.py --config wsj_biphone --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline"
timeout 900 $B > gpurun_out/bench_biphone.log 2>&1
LFMMI_OPTIONS=stream_ring=1 timeout 900 $B > gpurun_out/bench_biphone_ring.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
LFMMI_OPTIONS=stream_ring=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fb_stream_kernel" -s 1 -c 1 -o gpurun_out/prof_stream_ring python bench.py --config wsj_biphone --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_stream.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_sanitizers.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
