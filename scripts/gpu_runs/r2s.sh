mkdir -p gpurun_out
L=paper_2008_06134_b200
bash scripts/ab_variants.sh r2s_vote "base|$L/_sbrc.so|" "vote|$L/_sbrc_wv.so|" "base2|$L/_sbrc.so|" "vote2|$L/_sbrc_wv.so|"
for b in 8 0; do for f in fb none; do echo "band $b $f" >> gpurun_out/r2s_share.log; timeout 300 python scripts/rank_share.py $b hf $f >> gpurun_out/r2s_share.log 2>&1; done; done
