mkdir -p gpurun_out
for m in cone sbrc_shadow phong extinction none; do timeout 600 python scripts/full_parity.py 1 --mode $m >> gpurun_out/r5g_parity.log 2>&1; done
for m in cone shell none; do timeout 900 python scripts/full_parity.py 2 --mode $m >> gpurun_out/r5g_parity.log 2>&1; done
for m in shell phong extinction; do timeout 1200 python scripts/full_parity.py 3 --mode $m >> gpurun_out/r5g_parity.log 2>&1; done
timeout 1800 python scripts/full_parity.py 4 --mode shell >> gpurun_out/r5g_parity.log 2>&1
