mkdir -p gpurun_out
for v in "" l2r12 l2r16; do
LFMMI_LIB_VARIANT=$v timeout 600 python bench.py --config wsj_biphone --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/v_bi_$v.log 2>&1
LFMMI_LIB_VARIANT=$v timeout 900 python bench.py --config large --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/v_large_$v.log 2>&1
done
