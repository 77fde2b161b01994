mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_full_size_parity.py -q -p no:cacheprovider -x > gpurun_out/t_par.log 2>&1; echo "rc=$?" >> gpurun_out/t_par.log
timeout 1500 python -m pytest tests/test_sanitizers.py -q -p no:cacheprovider -k "ssplit or hmm or ring" > gpurun_out/t_san.log 2>&1; echo "rc=$?" >> gpurun_out/t_san.log
timeout 900 python bench.py --config wsj_biphone --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_bi.log 2>&1
for h in 30 36; do LFMMI_OPTIONS=split_h64=$h timeout 900 python bench.py --config wsj_biphone --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/bench_bi_h$h.log 2>&1; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fb_streamsplit -c 1 -o gpurun_out/prof_ss_src -f python bench.py --config wsj_biphone --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ss.log 2>&1
