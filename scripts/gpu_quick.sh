# quick: fused-kernel parity subset, ablation totals, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "configs or c2 or large or golden" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
: > gpurun_out/ablate.log
for ab in 0 1 3 63; do LFMMI_ABLATE=$ab python scripts/prof_sections.py 2>&1 | grep -E "TOTAL|ablate=" >> gpurun_out/ablate.log; done
LFMMI_DEBUG=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
