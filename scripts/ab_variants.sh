#!/bin/bash
# A/B the march kernel's launch-bounds variants: bash scripts/ab_variants.sh TAG lib1.so lib2.so ...
TAG=$1; shift
mkdir -p gpurun_out
for lib in "$@"; do
  echo "== $lib" >> gpurun_out/${TAG}_ab.log
  SBRC_LIB=$PWD/$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/${TAG}_ab.log 2>&1
done
echo done
