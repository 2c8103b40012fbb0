mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_frustum.py -x -q -s -p no:cacheprovider > gpurun_out/r2t_frustum_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_frustum_tests.log
timeout 900 python scripts/frustum_check.py 3 > gpurun_out/r2t_frustum_check.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_frustum_check.log
timeout 300 python scripts/pipeline_check.py > gpurun_out/r2t_pipe.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2t_pytest.log
