#!/bin/bash
# One GPU box round: gpu tests, bench, and (optionally) an ncu capture of the
# persistent AM kernel.  Usage (under gpurun): bash tools/gpu_round.sh TAG [ncu] [config]
TAG=${1:-dev}; NCU=${2:-}; CFG=${3:-c1}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -s 2>&1 | grep -E "stable|passed|failed|Error|error|assert" > gpurun_out/pytest_${TAG}.log
python bench.py --steps 20 --warmup 3 --config ${CFG} > gpurun_out/bench_${TAG}.log 2>&1
if [ -n "$NCU" ]; then
  python tools/profile_solve.py --config ${CFG} > gpurun_out/prof_plain_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:am_solve -s 1 -c 1 \
      -o gpurun_out/prof_${TAG} python tools/profile_solve.py --config ${CFG} > gpurun_out/ncu_${TAG}.log 2>&1
fi
tail -1 gpurun_out/pytest_${TAG}.log
