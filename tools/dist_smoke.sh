#!/bin/bash
# Multi-rank plumbing on a single-GPU box (under gpurun): bench.py under
# torchrun with 2 ranks sharing cuda:0, gloo for the collectives.  Not a
# scaling measurement (the ranks share one GPU).  Usage: bash tools/dist_smoke.sh TAG
TAG=${1:-dev}
mkdir -p gpurun_out
for sc in "c1 weak" "c1 strong" "c3 strong"; do
  set -- $sc
  BMPC_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --config $1 \
    --scaling $2 > gpurun_out/dist_${TAG}_$1_$2.log 2>&1
  echo "$1 $2 rc=$?"; tail -1 gpurun_out/dist_${TAG}_$1_$2.log | cut -c1-400
done
