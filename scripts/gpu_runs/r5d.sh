mkdir -p gpurun_out
timeout 600 python scripts/host_store_cost.py > gpurun_out/r5d_store.log 2>&1
timeout 600 python scripts/e2e_timeline.py > gpurun_out/r5d_timeline.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r5d_bench.log 2>&1
timeout 300 python scripts/image_hash.py 3 cone > gpurun_out/r5d_hash.log 2>&1
