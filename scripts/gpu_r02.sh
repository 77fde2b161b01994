mkdir -p gpurun_out
for nc in 68 70 72 74; do
LFMMI_OPTIONS=split_clusters=$nc timeout 600 python bench.py --config wsj_biphone --steps 10 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/nc_bi_$nc.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bi.csv python bench.py --config wsj_biphone --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
