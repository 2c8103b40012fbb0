mkdir -p gpurun_out
L=paper_2008_06134_b200
bash scripts/ab_variants.sh r3i "linear|$L/_sbrc.so|" "brick|$L/_sbrc_brick.so|" "linear2|$L/_sbrc.so|" "brick2|$L/_sbrc_brick.so|"
bash scripts/ab_variants.sh r3i_c2 "linear|$L/_sbrc.so|--config 2" "brick|$L/_sbrc_brick.so|--config 2"
bash scripts/ab_variants.sh r3i_c4 "linear|$L/_sbrc.so|--config 4" "brick|$L/_sbrc_brick.so|--config 4"
SBRC_LIB=$PWD/$L/_sbrc_brick.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3i_brick_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3i_brick_pytest.log
