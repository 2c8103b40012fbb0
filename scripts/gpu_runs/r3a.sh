mkdir -p gpurun_out
L=paper_2008_06134_b200
bash scripts/ab_variants.sh r3a "base|$L/_sbrc.so|" "pc3|$L/_sbrc_pc3.so|" "pc2|$L/_sbrc_pc2.so|" "tree|$L/_sbrc_ct.so|" "base2|$L/_sbrc.so|" "pc3b|$L/_sbrc_pc3.so|" "treeb|$L/_sbrc_ct.so|"
