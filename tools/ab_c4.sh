#!/bin/bash
# c4 (128-scene subset) timing of library variants in both precisions.
# Usage: bash tools/ab_c4.sh OUT v1 v2 ...   (prod = the product library)
OUT=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2109_10392_b200/_lib/libbatchmpc_b200.so
  [ "$v" != "prod" ] && lib=paper_2109_10392_b200/_lib/libbatchmpc_b200_$v.so
  for p in fp64 fp32; do
    echo "== $v c4 $p $(BMPC_LIB=$lib timeout 300 python tools/profile_solve.py --config c4 --scenes ${SCENES:-128} --reps 2 --precision $p 2>&1 | tail -1)"
  done
done > gpurun_out/$OUT 2>&1
cat gpurun_out/$OUT
