#!/bin/bash
# Time library variants (paper_2109_10392_b200/_lib/libbatchmpc_b200_<v>.so) on
# the BASELINE configs.  Usage (under gpurun): bash tools/variants.sh OUT v1 v2 ...
OUT=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2109_10392_b200/_lib/libbatchmpc_b200.so
  [ "$v" != "prod" ] && lib=paper_2109_10392_b200/_lib/libbatchmpc_b200_$v.so
  for c in ${CFGS:-c0 c1 c3 c4}; do
    echo "== $v $c"; BMPC_LIB=$lib python tools/profile_solve.py --config $c --reps 3 2>&1 | tail -1
  done
done > gpurun_out/$OUT 2>&1
