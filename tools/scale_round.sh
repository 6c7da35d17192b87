#!/bin/bash
# Bench lines for the larger BASELINE configs (no ncu: c4 runs for seconds).
mkdir -p gpurun_out
TAG=${1:-scale}
for cfg in c2 c3 c4; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_${cfg}.log 2>&1
done
