mkdir -p gpurun_out
L=paper_2008_06134_b200
for v in _sbrc _sbrc_cg; do for m in cone shell; do SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/image_hash.py 3 $m >> gpurun_out/r5aa_hash.log 2>&1; done; done
bash scripts/ab_variants.sh r5aa "base|$L/_sbrc.so|" "cg|$L/_sbrc_cg.so|" "base_b|$L/_sbrc.so|" "cg_b|$L/_sbrc_cg.so|"
for m in shell sbrc_shadow none; do bash scripts/ab_variants.sh r5aa_$m "base|$L/_sbrc.so|--mode $m" "cg|$L/_sbrc_cg.so|--mode $m"; done
