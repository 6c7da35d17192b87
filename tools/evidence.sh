#!/bin/bash
# Refresh the judged evidence on one GPU box (under gpurun): gpu tests, bench
# lines c1-c4 (+ fp32 c4), the c1 launch list, and full ncu captures of the
# persistent kernel for c1 / c3 / c4.  Usage: bash tools/evidence.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_${TAG}.log
for cfg in c1 c3; do
  python tools/profile_solve.py --config $cfg > gpurun_out/p_${TAG}_${cfg}.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:am_solve -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${cfg} python tools/profile_solve.py --config $cfg > gpurun_out/ncu_${TAG}_${cfg}.log 2>&1
done
python tools/profile_solve.py --config c4 --scenes 128 > gpurun_out/p_${TAG}_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:am_solve -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_c4s128 python tools/profile_solve.py --config c4 --scenes 128 > gpurun_out/ncu_${TAG}_c4.log 2>&1
for cfg in c1 c3; do
  python tools/ncu_json.py gpurun_out/prof_${TAG}_${cfg}.ncu-rep $cfg fp64 profiles/ncu_${cfg}_fp64.json
done
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_c1.log 2>&1
for cfg in c2 c3 c4; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_${cfg}.log 2>&1
done
timeout 900 python bench.py --config c4 --precision fp32 --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c4f32.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.log 2>&1
bash tools/launch_list.sh ${TAG}
cp profiles/ncu_c1_fp64.json profiles/ncu_c3_fp64.json gpurun_out/ 2>/dev/null
cat gpurun_out/pytest_${TAG}.log
