#!/bin/bash
# A/B of the obstacle culling (BMPC_CULL_MIN_M) on the BASELINE configs (c4: 128-scene subset).
OUT=${1:-ab_cull.txt}
mkdir -p gpurun_out
for c in c1 c2 c3 c4; do
  sc=""; [ $c = c4 ] && sc="--scenes 128"
  for mm in 1 1000; do
    echo "== cull_min_m=$mm $c"; BMPC_CULL_MIN_M=$mm timeout 300 python tools/profile_solve.py --config $c $sc --reps 3 2>&1 | tail -1
  done
done > gpurun_out/$OUT 2>&1
