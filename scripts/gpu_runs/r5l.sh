mkdir -p gpurun_out
L=paper_2008_06134_b200
for v in _sbrc _sbrc_lm3; do
  SBRC_LIB=$PWD/$L/$v.so timeout 1500 python scripts/frustum_check.py 3 > gpurun_out/r5l_frustum_c3$v.log 2>&1
done
