mkdir -p gpurun_out
timeout 1500 python scripts/frustum_check.py 3 > gpurun_out/r4m_frustum_c3.log 2>&1; echo rc=$? >> gpurun_out/r4m_frustum_c3.log
timeout 2400 python scripts/frustum_check.py 4 > gpurun_out/r4m_frustum_c4.log 2>&1; echo rc=$? >> gpurun_out/r4m_frustum_c4.log
