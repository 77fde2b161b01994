mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"linear_split_kernel<.int.16" -c 1 -o gpurun_out/prof_k16 -f python bench.py --config sweep --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k16.log 2>&1
