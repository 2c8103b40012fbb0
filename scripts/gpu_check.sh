#!/bin/bash
# One GPU-box session: parity tests, smoke, bench, and (optionally) ncu captures.
#   bash scripts/gpu_check.sh [tag] [ncu]     (run from the repo root under gpurun)
TAG=${1:-run}
NCU=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
if [ -n "$NCU" ]; then
  B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 300 $B > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"march_kernel|build_kernel" -c 2 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/${TAG}_plain.log
fi
echo done
