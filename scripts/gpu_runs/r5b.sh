mkdir -p gpurun_out
L=paper_2008_06134_b200
for rep in 1 2; do
for c in 3 2 4; do for v in _sbrc _sbrc_pf1 _sbrc_pf2 _sbrc_pf4 _sbrc_pf8; do
  SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/k1_time.py --config $c >> gpurun_out/r5b_k1.log 2>&1
done; done; done
bash scripts/ab_variants.sh r5b "pf0|$L/_sbrc.so|" "pf2|$L/_sbrc_pf2.so|" "pf4|$L/_sbrc_pf4.so|" "pf0b|$L/_sbrc.so|" "pf2b|$L/_sbrc_pf2.so|"
