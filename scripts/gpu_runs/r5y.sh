mkdir -p gpurun_out
L=paper_2008_06134_b200
for v in _sbrc _sbrc_late; do for m in cone shell sbrc_shadow; do SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/image_hash.py 3 $m >> gpurun_out/r5y_hash.log 2>&1; done; done
bash scripts/ab_variants.sh r5y "base|$L/_sbrc.so|" "late|$L/_sbrc_late.so|" "base_b|$L/_sbrc.so|" "late_b|$L/_sbrc_late.so|"
for m in shell sbrc_shadow; do bash scripts/ab_variants.sh r5y_$m "base|$L/_sbrc.so|--mode $m" "late|$L/_sbrc_late.so|--mode $m"; done
