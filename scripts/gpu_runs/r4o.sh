mkdir -p gpurun_out
L=paper_2008_06134_b200
bash scripts/ab_variants.sh r4o "mf0|$L/_sbrc_mf0.so|" "mf1|$L/_sbrc.so|" "mf0b|$L/_sbrc_mf0.so|" "mf1b|$L/_sbrc.so|"
bash scripts/ab_variants.sh r4o_none "mf0|$L/_sbrc_mf0.so|--mode none" "mf1|$L/_sbrc.so|--mode none"
bash scripts/ab_variants.sh r4o_shadow "mf0|$L/_sbrc_mf0.so|--mode sbrc_shadow" "mf1|$L/_sbrc.so|--mode sbrc_shadow"
for l in _sbrc_mf0 _sbrc; do for m in cone none; do SBRC_LIB=$PWD/$L/$l.so timeout 300 python scripts/image_hash.py 3 $m >> gpurun_out/r4o_hash.log 2>&1; done; done
