mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "configs or large or packed" > gpurun_out/pytest_stream.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_stream.log
: > gpurun_out/configs.log
for m in 1024x1 512x2 1024x2; do
  for c in wsj_biphone large; do
    LFMMI_STREAM_MODE=$m timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$m.log 2>&1; echo "$c $m rc=$?" >> gpurun_out/configs.log
  done
done
