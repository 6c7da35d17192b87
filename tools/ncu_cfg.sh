#!/bin/bash
# One full ncu capture of the persistent AM kernel per config (under gpurun),
# each only after the same command ran clean without ncu; JSON summaries for
# bench.py's roofline block.  Usage: bash tools/ncu_cfg.sh TAG cfg1 [cfg2 ...]
TAG=$1; shift
mkdir -p gpurun_out
for cfg in "$@"; do
  extra=""
  [ "${cfg%f32}" != "$cfg" ] && extra="--precision fp32"
  base=${cfg%f32}
  timeout 600 python tools/profile_solve.py --config $base $extra > gpurun_out/p_${TAG}_${cfg}.log 2>&1 || { echo "$cfg plain run failed"; continue; }
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:am_solve -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${cfg} python tools/profile_solve.py --config $base $extra > gpurun_out/ncu_${TAG}_${cfg}.log 2>&1
  prec=fp64; [ -n "$extra" ] && prec=fp32
  python tools/ncu_json.py gpurun_out/prof_${TAG}_${cfg}.ncu-rep $base $prec gpurun_out/ncu_${base}_${prec}.json > /dev/null && echo "$cfg ok"
done
