#!/bin/bash
# A/B the c1 step (tools/step_breakdown.py) across library variants on one box.
# Usage (under gpurun): bash tools/ab_step.sh v1 v2 ...   ("prod" = the product library)
for r in 1 2; do for v in "$@"; do
  lib=paper_2109_10392_b200/_lib/libbatchmpc_b200.so
  [ "$v" != "prod" ] && lib=paper_2109_10392_b200/_lib/libbatchmpc_b200_$v.so
  echo "== $v"; BMPC_LIB=$lib python tools/step_breakdown.py ${CFG:-c1} 2>&1 | tail -3
done; done
