mkdir -p gpurun_out
for l in _sbrc _sbrc_g2 _sbrc_g4w _sbrc_lat2; do
  echo "== $l" >> gpurun_out/r3d_share.log
  SBRC_LIB=$PWD/paper_2008_06134_b200/$l.so timeout 900 python scripts/frustum_check.py 3 >> gpurun_out/r3d_share.log 2>&1
done
