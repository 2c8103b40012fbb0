mkdir -p gpurun_out
for c in 3 2 4; do for l in _sbrc _sbrc_u1m6 _sbrc_u1m7 _sbrc_u1m8 _sbrc; do
  SBRC_LIB=$PWD/paper_2008_06134_b200/$l.so timeout 600 python scripts/k1_time.py --config $c >> gpurun_out/r3h_k1ab.log 2>&1
done; done
