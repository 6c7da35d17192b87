#!/bin/bash
# A/B of a library variant against the product library (under gpurun): bitwise
# comparison of the solve on golden fixtures, then timings on BASELINE configs.
# Usage: bash tools/ab_variant.sh OUT VARIANT [VARIANT...]; CFGS / BITS override the lists,
# PREC=fp32 runs the fp32 mode, ARGS adds profile_solve.py arguments.
OUT=$1; shift
mkdir -p gpurun_out
L=paper_2109_10392_b200/_lib
{
for v in "$@"; do
  for g in ${BITS:-c1 c2f c3f c4f}; do
    BMPC_LIB=$L/libbatchmpc_b200.so python tools/bits_dump.py $g /tmp/bits_prod_$g.npz > /dev/null 2>&1
    BMPC_LIB=$L/libbatchmpc_b200_$v.so python tools/bits_dump.py $g /tmp/bits_${v}_$g.npz > /dev/null 2>&1
    python - <<PY
import numpy as np
a, b = np.load("/tmp/bits_prod_$g.npz"), np.load("/tmp/bits_${v}_$g.npz")
same = all(np.array_equal(a[k].view(np.int64), b[k].view(np.int64)) for k in ("c_x", "c_y", "c_psi"))
d = max(float(np.abs(a[k] - b[k]).max()) for k in ("c_x", "c_y", "c_psi"))
print("bits $v $g:", "IDENTICAL" if same else f"DIFFER max abs {d:.3e}")
PY
  done
done
for v in prod "$@"; do
  lib=$L/libbatchmpc_b200.so
  [ "$v" != "prod" ] && lib=$L/libbatchmpc_b200_$v.so
  for c in ${CFGS:-c1 c2 c3}; do
    echo "== $v $c $(BMPC_LIB=$lib timeout 600 python tools/profile_solve.py --config $c --reps ${REPS:-3} ${PREC:+--precision $PREC} $ARGS 2>&1 | tail -1)"
  done
done
} > gpurun_out/$OUT 2>&1
cat gpurun_out/$OUT
