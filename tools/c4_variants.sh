#!/bin/bash
# c4 (128-scene subset) timing of library variants.  Usage: bash tools/c4_variants.sh OUT v1 v2 ...
OUT=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2109_10392_b200/_lib/libbatchmpc_b200.so
  [ "$v" != "prod" ] && lib=paper_2109_10392_b200/_lib/libbatchmpc_b200_$v.so
  echo "== $v"; BMPC_LIB=$lib timeout 300 python tools/profile_solve.py --config c4 --scenes 128 --reps 3 2>&1 | tail -1
done > gpurun_out/$OUT 2>&1
