#!/bin/bash
# Launch list of the bench command (per-kernel device times, cold-cache/serialised
# under ncu -- compare shares, not absolutes).  Run under gpurun.
mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/launch_plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/launch_ncu_${TAG}.log 2>&1
