# ncu captures only (den + num kernels) for the current build
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_tile_kernel<float, .int.512" -s 2 -c 1 -o gpurun_out/prof_den python bench.py --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_den.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fb_tile_kernel<float, .int.32," -s 2 -c 1 -o gpurun_out/prof_num python bench.py --profile --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_num.log 2>&1
