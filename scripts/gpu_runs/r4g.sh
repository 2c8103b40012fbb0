mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r4g_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r4g_bench.log
timeout 1200 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r4g_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r4g_ref.log
