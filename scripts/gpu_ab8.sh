mkdir -p gpurun_out; : > gpurun_out/ab8.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
one() { env $2 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$1', 'ms/step', round(d['ms_per_step'], 4), 'den', round(d['roofline']['launch_ms'], 4), 'value', round(d['value']/1e6, 3))" >> gpurun_out/ab8.log; }
for r in 1 2; do for b in 12 16 20; do one bias$b "LFMMI_CHORE_BIAS=$b"; done; done
timeout 300 python scripts/time_passes.py wsj_mono > gpurun_out/passes.log 2>&1
