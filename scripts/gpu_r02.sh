# round-2: sweep128 (N=8 per-rank proxy): numerator launch shape x den cluster count
mkdir -p gpurun_out
S="python bench.py --config sweep --batch 128 --steps 5 --warmup 3 --no-extra-e2e --no-cpu-baseline"
for k16 in 1 0; do for nc in 71 68 64 60 56; do LFMMI_OPTIONS=linear_k16=$k16,split_clusters=$nc timeout 600 $S > gpurun_out/sw128_k${k16}_nc$nc.log 2>&1; done; done
W="python bench.py --steps 20 --warmup 3 --no-extra-e2e --no-cpu-baseline"
for h in 31 32 33 34; do LFMMI_OPTIONS=split_h64=$h timeout 600 $W > gpurun_out/wsj_h$h.log 2>&1; done
for cb in 4 8 16; do LFMMI_OPTIONS=chore_bias=$cb timeout 600 $W > gpurun_out/wsj_cb$cb.log 2>&1; done
timeout 900 python bench.py --config sweep --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/sweep.log 2>&1
LFMMI_OPTIONS=linear_k16=0 timeout 900 python bench.py --config sweep --steps 3 --warmup 3 --no-extra-e2e --no-cpu-baseline > gpurun_out/sweep_k16sep.log 2>&1
