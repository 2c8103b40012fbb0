mkdir -p gpurun_out
timeout 900 python scripts/frustum_check.py 3 > gpurun_out/r4b_frustum_c3.log 2>&1; echo rc=$? >> gpurun_out/r4b_frustum_c3.log
bash scripts/multirank_flow.sh r4b
