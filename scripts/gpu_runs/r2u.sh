mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_frustum.py -x -q -s -p no:cacheprovider > gpurun_out/r2u_frustum_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_frustum_tests.log
timeout 1200 python scripts/frustum_check.py 3 > gpurun_out/r2u_frustum_check.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_frustum_check.log
