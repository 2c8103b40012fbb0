mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"march_kernel|build_kernel" -c 2 -o gpurun_out/prof_r01 $B > gpurun_out/ncu_full.log 2>&1
echo rc=$?
