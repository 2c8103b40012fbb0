mkdir -p gpurun_out
L=paper_2008_06134_b200
for v in _sbrc _sbrc_bulk; do
  SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/image_hash.py 3 cone >> gpurun_out/r5f_hash.log 2>&1
  SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/image_hash.py 1 shell >> gpurun_out/r5f_hash.log 2>&1
  SBRC_LIB=$PWD/$L/$v.so timeout 300 python scripts/host_store_cost.py 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/r5f_store.log
done
for v in _sbrc _sbrc_bulk _sbrc _sbrc_bulk; do
  SBRC_LIB=$PWD/$L/$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-full-frame 2>&1 | grep "^{" | sed "s/^/$v /" >> gpurun_out/r5f_bench.log
done
