mkdir -p gpurun_out
bash scripts/ab_variants.sh r4r "cone|paper_2008_06134_b200/_sbrc.so|" "shell|paper_2008_06134_b200/_sbrc.so|--mode shell" "shadow|paper_2008_06134_b200/_sbrc.so|--mode sbrc_shadow"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r4r_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r4r_pytest.log
for m in cone shell; do timeout 300 python scripts/image_hash.py 3 $m >> gpurun_out/r4r_hash.log 2>&1; done
