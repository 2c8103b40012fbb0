mkdir -p gpurun_out
for c in 3 2 4; do for l in _sbrc_fs0 _sbrc _sbrc_fs0 _sbrc; do
  SBRC_LIB=$PWD/paper_2008_06134_b200/$l.so timeout 600 python scripts/k1_time.py --config $c >> gpurun_out/r4n_k1ab.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "build or parity or sparse or frustum or scale" > gpurun_out/r4n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r4n_pytest.log
