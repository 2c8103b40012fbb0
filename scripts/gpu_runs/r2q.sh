mkdir -p gpurun_out
for m in cone shell; do
L=paper_2008_06134_b200
bash scripts/ab_variants.sh r2q_$m "pk0|$L/_sbrc_pk0.so|--mode $m" "pk1|$L/_sbrc_pk1.so|--mode $m" "pk2|$L/_sbrc_pk2.so|--mode $m" "pk3|$L/_sbrc_pk3.so|--mode $m"
done
