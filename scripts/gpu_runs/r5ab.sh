mkdir -p gpurun_out
L=paper_2008_06134_b200
for c in 3 2 4; do for v in _sbrc _sbrc_r2 _sbrc_r8 _sbrc_r16; do
  SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/k1_time.py --config $c >> gpurun_out/r5ab_k1.log 2>&1
done; done
