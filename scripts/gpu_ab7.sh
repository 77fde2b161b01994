mkdir -p gpurun_out; : > gpurun_out/ab7.log
one() { env $2 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$1', 'ms/step', round(d['ms_per_step'], 4), 'den', round(d['roofline']['launch_ms'], 4), 'value', round(d['value']/1e6, 3))" >> gpurun_out/ab7.log; }
for b in 8 12 16 24; do one bias$b-f100 "LFMMI_CHORE_BIAS=$b"; done
for f in 50 150 200; do one bias12-f$f "LFMMI_CHORE_BIAS=12 LFMMI_FLUSH_BIAS_PCT=$f"; done
for b in 8 12 16 24; do one bias$b-f100 "LFMMI_CHORE_BIAS=$b"; done
