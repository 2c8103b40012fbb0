mkdir -p gpurun_out
timeout 1500 python scripts/frustum_check.py 3 > gpurun_out/r4t_frustum_c3.log 2>&1
timeout 2400 python scripts/frustum_check.py 4 > gpurun_out/r4t_frustum_c4.log 2>&1
timeout 600 python scripts/pipeline_check.py 3 > gpurun_out/r4t_pipe_c3.log 2>&1
timeout 1500 python scripts/pipeline_check.py 4 > gpurun_out/r4t_pipe_c4.log 2>&1
