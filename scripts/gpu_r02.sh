mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_sanitizers.py > gpurun_out/t_all.log 2>&1; echo "rc=$?" >> gpurun_out/t_all.log
timeout 600 python bench.py --config toy --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_toy.log 2>&1
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
