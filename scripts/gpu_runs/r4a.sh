mkdir -p gpurun_out
bash scripts/gpu_check.sh r4a ncu
for c in 1 2 4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-full-frame > gpurun_out/r4a_bench_c$c.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_bench_c$c.log; done
timeout 1500 python bench.py --config 5 --warmup 3 > gpurun_out/r4a_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_c5.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r4a_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_ref.log
