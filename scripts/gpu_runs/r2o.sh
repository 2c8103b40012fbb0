mkdir -p gpurun_out
for c in 3 2; do for l in _sbrc_k1A0 _sbrc _sbrc_k1A3 _sbrc_k1A6 _sbrc_k1A3M8; do
  SBRC_LIB=$PWD/paper_2008_06134_b200/$l.so timeout 300 python scripts/k1_time.py --config $c >> gpurun_out/r2o_k1ab.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2o_pytest.log
