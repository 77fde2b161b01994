# bench every BASELINE config on one GPU (+ the reference arm, bounded samples)
mkdir -p gpurun_out; : > gpurun_out/configs.log
for c in toy wsj_mono wsj_biphone large sweep; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?" >> gpurun_out/configs.log
  timeout 600 python bench.py --config $c --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$c.log 2>&1; echo "$c ref rc=$?" >> gpurun_out/configs.log
done
