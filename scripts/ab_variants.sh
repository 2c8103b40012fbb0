#!/bin/bash
# A/B bench variants: bash scripts/ab_variants.sh TAG "label|lib.so|bench args" ...
TAG=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  IFS='|' read -r label lib args <<< "$spec"
  echo "== $label" >> gpurun_out/${TAG}_ab.log
  SBRC_LIB=$PWD/$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args >> gpurun_out/${TAG}_ab.log 2>&1
done
echo done
