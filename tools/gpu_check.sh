#!/bin/bash
# Quick GPU check (under gpurun): the whole -m gpu suite (no -x, failures
# listed), smoke(), then the c1 bench line.  Usage: bash tools/gpu_check.sh TAG [pytest -k expr]
TAG=${1:-dev}; K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf -s -k "$K" > gpurun_out/pytest_${TAG}.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -rf -s > gpurun_out/pytest_${TAG}.log 2>&1
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1
tail -3 gpurun_out/pytest_${TAG}.log; tail -1 gpurun_out/smoke_${TAG}.log
python tools/show_bench.py gpurun_out/bench_${TAG}.log 2>/dev/null | head -5
