#!/bin/bash
# Judged evidence for round 2 (under gpurun): gpu tests, ncu captures of the
# persistent kernel per config (JSON summaries into profiles/ before the bench
# lines read them), bench lines c1-c4 (+ c4 fp32), the reference arm, the c1
# launch list.  Usage: bash tools/evidence_r02.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out profiles
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_${TAG}.log 2>&1
tail -2 gpurun_out/pytest_${TAG}.log
# NONCU=1: skip the ncu captures (the persistent kernel unchanged since the last ones)
[ -n "$NONCU" ] || for spec in "c1::" "c2::" "c3::" "c4:--scenes 128:subset: 128 of the 1024 c4 scenes (a full-c4 capture does not finish under ncu replay)" \
            "c4f32:--scenes 128 --precision fp32:subset: 128 of the 1024 c4 scenes, fp32 mode" \
            "c1f32:--precision fp32:fp32 mode" "c3f32:--precision fp32:fp32 mode"; do
  cfg=${spec%%:*}; rest=${spec#*:}; args=${rest%%:*}; note=${rest#*:}
  base=${cfg%f32}; prec=fp64; [ "$base" != "$cfg" ] && prec=fp32
  timeout 600 python tools/profile_solve.py --config $base $args > gpurun_out/p_${TAG}_${cfg}.log 2>&1 || { echo "$cfg plain failed"; continue; }
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:am_solve -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${cfg} python tools/profile_solve.py --config $base $args > gpurun_out/ncu_${TAG}_${cfg}.log 2>&1
  python tools/ncu_json.py gpurun_out/prof_${TAG}_${cfg}.ncu-rep $base $prec profiles/ncu_${base}_${prec}.json "$note" > /dev/null \
    && cp profiles/ncu_${base}_${prec}.json gpurun_out/ && echo "ncu $cfg ok"
  # small text summaries travel back; the reports themselves only for c1 (the
  # merge back is capped at 64 MiB)
  ncu -i gpurun_out/prof_${TAG}_${cfg}.ncu-rep --page details > gpurun_out/${TAG}_${cfg}_ncu.txt 2>&1
  python tools/ncu_srclines.py gpurun_out/prof_${TAG}_${cfg}.ncu-rep 60 > gpurun_out/${TAG}_${cfg}_ncu_lines.txt 2>&1
  [ "$cfg" != "c1" ] && rm -f gpurun_out/prof_${TAG}_${cfg}.ncu-rep
done
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_c1.log 2>&1
for cfg in c2 c3 c4; do
  timeout 1200 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_${cfg}.log 2>&1
done
timeout 1200 python bench.py --config c4 --precision fp32 --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c4f32.log 2>&1
timeout 600 python bench.py --precision fp32 --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_c1f32.log 2>&1
timeout 900 python bench.py --config c3 --precision fp32 --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c3f32.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.log 2>&1
bash tools/launch_list.sh ${TAG}
for f in gpurun_out/bench_${TAG}_*.log; do tail -1 $f | cut -c1-160; done
du -sh gpurun_out
