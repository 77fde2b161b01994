mkdir -p gpurun_out
for o in "emit=1" "emit=0"; do
LFMMI_OPTIONS=$o timeout 600 python bench.py --config wsj_biphone --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/em_bi_$o.log 2>&1
LFMMI_OPTIONS=$o timeout 900 python bench.py --config large --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/em_large_$o.log 2>&1
done
