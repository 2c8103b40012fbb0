mkdir -p gpurun_out
L=paper_2008_06134_b200
for v in _sbrc _sbrc_pfall _sbrc_pfnone; do for m in cone none phong extinction; do SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/image_hash.py 3 $m >> gpurun_out/r5i_hash.log 2>&1; done; done
for m in cone none phong extinction; do bash scripts/ab_variants.sh r5i_$m "default|$L/_sbrc.so|--mode $m" "pf_always|$L/_sbrc_pfall.so|--mode $m" "pf_never|$L/_sbrc_pfnone.so|--mode $m"; done
bash scripts/ab_variants.sh r5i_c2none "default|$L/_sbrc.so|--config 2 --mode none" "pf_always|$L/_sbrc_pfall.so|--config 2 --mode none"
bash scripts/ab_variants.sh r5i_c4none "default|$L/_sbrc.so|--config 4 --mode none" "pf_always|$L/_sbrc_pfall.so|--config 4 --mode none"
