#!/bin/bash
# Split-kernel bring-up: parity tests, pass timings, bench (WSJ-mono).
mkdir -p gpurun_out
LFMMI_DEBUG=1 timeout 300 python scripts/time_passes.py wsj_mono > gpurun_out/split_passes.log 2>&1
echo "passes rc=$?"
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/split_pytest.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/split_pytest.log
grep -v Warning gpurun_out/split_passes.log | grep -v "^  t(" | tail -12
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/split_bench.log 2>&1
echo "bench rc=$?"; grep -o '"value": [0-9.]*\|"ms_per_step": [0-9.]*' gpurun_out/split_bench.log | head -3
