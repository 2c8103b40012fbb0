mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r2w_gpu.txt 2>&1
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/r2w_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_bench.log
for c in 1 2 4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-full-frame > gpurun_out/r2w_bench_c$c.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_bench_c$c.log; done
timeout 1500 python bench.py --config 5 --warmup 3 > gpurun_out/r2w_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_c5.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2w_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_ref.log
timeout 1500 python scripts/frustum_check.py 4 > gpurun_out/r2w_frustum_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_frustum_c4.log
