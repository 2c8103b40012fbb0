mkdir -p gpurun_out
L=paper_2008_06134_b200
for m in cone shell sbrc_shadow; do
bash scripts/ab_variants.sh r3j_$m "quads|$L/_sbrc.so|--mode $m" "pairs|$L/_sbrc_pairs.so|--mode $m" "quads2|$L/_sbrc.so|--mode $m" "pairs2|$L/_sbrc_pairs.so|--mode $m"
for l in _sbrc _sbrc_pairs; do SBRC_LIB=$PWD/$L/$l.so timeout 300 python scripts/image_hash.py 3 $m >> gpurun_out/r3j_hash.log 2>&1; done
done
