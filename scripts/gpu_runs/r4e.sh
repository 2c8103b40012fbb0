mkdir -p gpurun_out
timeout 1500 python scripts/frustum_check.py 3 > gpurun_out/r4e_frustum_c3.log 2>&1; echo rc=$? >> gpurun_out/r4e_frustum_c3.log
timeout 1500 python scripts/frustum_check.py 3 > gpurun_out/r4e_frustum_c3b.log 2>&1; echo rc=$? >> gpurun_out/r4e_frustum_c3b.log
bash scripts/multirank_flow.sh r4e
