mkdir -p gpurun_out
L=paper_2008_06134_b200
bash scripts/ab_variants.sh r4p "lf0|$L/_sbrc_lf0.so|" "lf1|$L/_sbrc.so|" "lf0b|$L/_sbrc_lf0.so|" "lf1b|$L/_sbrc.so|"
bash scripts/ab_variants.sh r4p_shell "lf0|$L/_sbrc_lf0.so|--mode shell" "lf1|$L/_sbrc.so|--mode shell"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r4p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r4p_pytest.log
