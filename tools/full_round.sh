#!/bin/bash
# Round-end evidence on one GPU box: gpu tests, bench lines for every config,
# the c1 launch list, and full ncu captures of c3/c4 (for profiles/ncu_*.json).
TAG=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_${TAG}.log
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_c1.log 2>&1
for cfg in c2 c3 c4; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_${cfg}.log 2>&1
done
timeout 900 python bench.py --config c4 --precision fp32 --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c4f32.log 2>&1
bash tools/launch_list.sh ${TAG}
for cfg in c3 c4; do
  python tools/profile_solve.py --config $cfg > gpurun_out/p_${TAG}_${cfg}.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:am_solve -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${cfg} python tools/profile_solve.py --config $cfg > gpurun_out/ncu_${TAG}_${cfg}.log 2>&1
done
