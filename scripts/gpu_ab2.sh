# A/B: fused vs two-pass, alternating on the same box, plus e2e
mkdir -p gpurun_out; : > gpurun_out/ab2.log
one() { env $2 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$1', 'ms/step', round(d['ms_per_step'], 4), 'value', round(d['value']/1e6, 3), 'e2e', round(d['e2e']['value']/1e6, 3), d['e2e']['ms_per_step'], 'launches', d['gpu_launches'])" >> gpurun_out/ab2.log; }
for r in 1 2; do one twopass ""; one fused "LFMMI_FUSED=1"; done
