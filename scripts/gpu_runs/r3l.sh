mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3l_pytest.log
for c in 2 3; do timeout 600 python bench.py --config $c --mode sbrc_shadow --steps 30 --warmup 5 --no-cpu-baseline --no-full-frame --no-e2e > gpurun_out/r3l_shadow_c$c.log 2>&1; done
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-full-frame > gpurun_out/r3l_bench.log 2>&1
