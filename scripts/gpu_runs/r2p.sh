mkdir -p gpurun_out
for m in cone shell sbrc_shadow; do
bash scripts/ab_variants.sh r2p_$m "pk0|paper_2008_06134_b200/_sbrc_pk0.so|--mode $m" "pk1|paper_2008_06134_b200/_sbrc.so|--mode $m" "pk0b|paper_2008_06134_b200/_sbrc_pk0.so|--mode $m" "pk1b|paper_2008_06134_b200/_sbrc.so|--mode $m"
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2p_pytest.log
