#!/bin/bash
# round evidence: full bench line (with the CPU baseline), launch list of one
# solve, ncu --set full of the dominant kernel (first launch = finest level)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -c 2500 gpurun_out/bench_full.json
PROF_SOLVES=1 timeout 300 python tools/profile_solve.py > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/profile_solve.py > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
PROF_SOLVES=1 PROF_MAXIT=1 timeout 300 python tools/profile_solve.py > gpurun_out/plain2.log 2>&1 && \
  PROF_SOLVES=1 PROF_MAXIT=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"$1" -c 1 -o gpurun_out/dom -f python tools/profile_solve.py > gpurun_out/ncu_dom.log 2>&1
echo "ncu dom exit $?"
