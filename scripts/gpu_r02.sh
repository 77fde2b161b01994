mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_full_size_parity.py -q -p no:cacheprovider -k "hmm" > gpurun_out/t_hmm.log 2>&1; echo "rc=$?" >> gpurun_out/t_hmm.log
LFMMI_OPTIONS=small_arcs=0 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/t_small0.log 2>&1; echo "rc=$?" >> gpurun_out/t_small0.log
timeout 900 python bench.py --config hmm --steps 20 --warmup 3 --no-extra-e2e > gpurun_out/bench_hmm.log 2>&1
LFMMI_OPTIONS=split=0 timeout 900 python bench.py --config hmm --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_hmm_tile.log 2>&1
LFMMI_OPTIONS=small_arcs=100000 timeout 900 python bench.py --config hmm --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_hmm_old.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hmm.csv python bench.py --config hmm --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
