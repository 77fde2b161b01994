mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_sanitizers.py > gpurun_out/t_all.log 2>&1; echo "rc=$?" >> gpurun_out/t_all.log
timeout 1500 python -m pytest tests/test_sanitizers.py -q -p no:cacheprovider -k "ssplit or ring or stream" > gpurun_out/t_san.log 2>&1; echo "rc=$?" >> gpurun_out/t_san.log
timeout 600 python bench.py --config wsj_biphone --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_bi.log 2>&1
timeout 900 python bench.py --config large --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_large.log 2>&1
