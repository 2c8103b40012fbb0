mkdir -p gpurun_out
./scripts/tma_probe.bin > gpurun_out/r2z_probe.log 2>&1; echo rc=$? >> gpurun_out/r2z_probe.log
for c in 3 2; do for l in _sbrc_k1T0 _sbrc _sbrc_k1T70 _sbrc_k1T200; do
  SBRC_LIB=$PWD/paper_2008_06134_b200/$l.so timeout 300 python scripts/k1_time.py --config $c >> gpurun_out/r2z_k1ab.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2z_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2z_pytest.log
