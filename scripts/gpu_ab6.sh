mkdir -p gpurun_out; : > gpurun_out/ab6.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "configs or c2 or golden or packed or nan" > gpurun_out/pytest_ab6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab6.log
for r in 1 2 3; do timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'], 4), 'den', round(d['roofline']['launch_ms'], 4), 'value', round(d['value']/1e6, 3))" >> gpurun_out/ab6.log; done
