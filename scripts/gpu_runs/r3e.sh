mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_frustum.py -x -q -p no:cacheprovider > gpurun_out/r3e_tests.log 2>&1; echo rc=$? >> gpurun_out/r3e_tests.log
timeout 900 python scripts/frustum_check.py 3 > gpurun_out/r3e_frustum_c3.log 2>&1; echo rc=$? >> gpurun_out/r3e_frustum_c3.log
timeout 1800 python scripts/frustum_check.py 4 > gpurun_out/r3e_frustum_c4.log 2>&1; echo rc=$? >> gpurun_out/r3e_frustum_c4.log
