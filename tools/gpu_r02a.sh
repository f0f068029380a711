#!/bin/bash
# r02 pass A: GPU tests, the new default bench line (configs[2]), launch list
# of two 513^3 wedge iterations, ncu --set full of the 513^3 Jacobi sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -c 3000 gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
PROF_SOLVES=1 PROF_MAXIT=2 timeout 300 python tools/profile_solve.py > gpurun_out/plain.log 2>&1 && \
  PROF_SOLVES=1 PROF_MAXIT=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python tools/profile_solve.py > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
PROF_SOLVES=1 PROF_MAXIT=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_stencil" -c 3 -o gpurun_out/dom_c2 -f python tools/profile_solve.py > gpurun_out/ncu_dom.log 2>&1
echo "ncu dom exit $?"
