mkdir -p gpurun_out
L=paper_2008_06134_b200
for v in _sbrc _sbrc_npf4 _sbrc_npf5 _sbrc_npf6; do for m in cone shell none sbrc_shadow; do SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/image_hash.py 3 $m >> gpurun_out/r5h_hash.log 2>&1; done; done
bash scripts/ab_variants.sh r5h "pf|$L/_sbrc.so|" "npf4|$L/_sbrc_npf4.so|" "npf5|$L/_sbrc_npf5.so|" "npf6|$L/_sbrc_npf6.so|" "pf_b|$L/_sbrc.so|" "npf5_b|$L/_sbrc_npf5.so|"
for m in shell none sbrc_shadow; do bash scripts/ab_variants.sh r5h_$m "pf|$L/_sbrc.so|--mode $m" "npf4|$L/_sbrc_npf4.so|--mode $m" "npf5|$L/_sbrc_npf5.so|--mode $m"; done
bash scripts/ab_variants.sh r5h_c2 "pf|$L/_sbrc.so|--config 2" "npf5|$L/_sbrc_npf5.so|--config 2"
bash scripts/ab_variants.sh r5h_c1 "pf|$L/_sbrc.so|--config 1" "npf5|$L/_sbrc_npf5.so|--config 1"
