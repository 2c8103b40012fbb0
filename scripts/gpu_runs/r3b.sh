mkdir -p gpurun_out
SBRC_LIB=$PWD/paper_2008_06134_b200/_sbrc_checked.so timeout 900 python scripts/checked_run.py > gpurun_out/r3b_checked.log 2>&1; echo rc=$? >> gpurun_out/r3b_checked.log
timeout 1800 python scripts/frustum_check.py 4 > gpurun_out/r3b_frustum_c4.log 2>&1; echo rc=$? >> gpurun_out/r3b_frustum_c4.log
