#!/bin/bash
# Control-flow check of the multi-rank bench on a ONE-GPU box: 2 ranks under
# torchrun, both on cuda:0, gloo instead of NCCL (NCCL needs distinct GPUs).
# Exercises rank setup, p2p/NCCL-path assembly, the frustum calibration
# (choose_march_kernel + rebalance), pipelining and the JSON line; the
# timings of such a run mean nothing.   bash scripts/multirank_flow.sh TAG
TAG=${1:-flow}
mkdir -p gpurun_out
export SBRC_BENCH_SAME_GPU=1 SBRC_BENCH_BACKEND=gloo
for cfg in 1 3; do for b in frustum replicated; do for asm in p2p nccl; do
  echo "== config $cfg build $b assemble $asm" >> gpurun_out/${TAG}_flow.log
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --config $cfg --steps 3 --warmup 3 \
    --build $b --assemble $asm --no-cpu-baseline --no-full-frame >> gpurun_out/${TAG}_flow.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_flow.log
done; done; done
