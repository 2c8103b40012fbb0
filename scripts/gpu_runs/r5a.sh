mkdir -p gpurun_out
L=paper_2008_06134_b200
for v in _sbrc _sbrc_nw2 _sbrc_nw6 _sbrc_nw2b; do for m in cone shell; do SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/image_hash.py 3 $m | sed "s/^/$v /" >> gpurun_out/r5a_hash.log 2>&1; done; done
bash scripts/ab_variants.sh r5a "nw4|$L/_sbrc.so|" "nw2|$L/_sbrc_nw2.so|" "nw6|$L/_sbrc_nw6.so|" "nw2b|$L/_sbrc_nw2b.so|" "nw4b|$L/_sbrc.so|" "nw2c|$L/_sbrc_nw2.so|"
bash scripts/ab_variants.sh r5a_shell "nw4|$L/_sbrc.so|--mode shell" "nw2|$L/_sbrc_nw2.so|--mode shell" "nw6|$L/_sbrc_nw6.so|--mode shell" "nw2b|$L/_sbrc_nw2b.so|--mode shell"
