#!/bin/bash
# one GPU call: gpu tests, bench, large-config solves, then ncu --set full on the solve kernels
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
for c in "wedge3 --n 257" "cube --n 257" "wedge3 --n 513"; do
  timeout 600 python tools/run_config.py $c >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
done
cat gpurun_out/configs.jsonl
PROF_SOLVES=1 PROF_MAXIT=2 timeout 300 python tools/profile_solve.py > gpurun_out/plain.log 2>&1 && \
PROF_SOLVES=1 PROF_MAXIT=2 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'k_stencil|k_corr|k_restrict2|k_bcg|k_fdm' -c 60 -o gpurun_out/prof -f python tools/profile_solve.py > gpurun_out/ncu.log 2>&1
echo ncu exit $?
