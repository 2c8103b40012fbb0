mkdir -p gpurun_out
timeout 1500 python scripts/full_parity.py 1 2 3 > gpurun_out/r4f_full_parity.log 2>&1
timeout 900 python scripts/full_parity.py 3 --mode none >> gpurun_out/r4f_full_parity.log 2>&1
timeout 900 python scripts/full_parity.py 3 --mode sbrc_shadow >> gpurun_out/r4f_full_parity.log 2>&1
nproc >> gpurun_out/r4f_full_parity.log
