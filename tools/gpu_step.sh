#!/bin/bash
# bench line + launch list of two 513^3 iterations (cold, serialised: compare shares)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err; tail -c 300 gpurun_out/bench_step.json; tail -3 gpurun_out/bench_step.err
PROF_CONFIG=c2 PROF_SOLVES=1 PROF_MAXIT=2 timeout -s KILL 200 python tools/profile_solve.py > gpurun_out/plain.log 2>&1 && \
  PROF_CONFIG=c2 PROF_SOLVES=1 PROF_MAXIT=2 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python tools/profile_solve.py > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
