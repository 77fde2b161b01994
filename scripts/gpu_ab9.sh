mkdir -p gpurun_out; : > gpurun_out/ab9.log
one() { env $2 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$1', 'ms/step', round(d['ms_per_step'], 4), 'den', round(d['roofline']['launch_ms'], 4), 'value', round(d['value']/1e6, 3))" >> gpurun_out/ab9.log; }
one base ""
for bb in 8 12 24 32; do one bwd$bb "LFMMI_CHORE_BIAS_BWD=$bb"; done
for f in 50 150 200 300; do one flush$f "LFMMI_FLUSH_BIAS_PCT=$f"; done
for fw in 12 20 24; do one fwd$fw "LFMMI_CHORE_BIAS=$fw LFMMI_CHORE_BIAS_BWD=16"; done
one base ""
