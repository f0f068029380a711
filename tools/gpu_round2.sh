#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/live_breakdown.py gpurun_out/live_129.txt > /dev/null 2>gpurun_out/live.err; cat gpurun_out/live_129.txt | head -40
timeout 300 python tools/kernel_table_at.py 257 > gpurun_out/kt257.json 2>>gpurun_out/kt.err; cat gpurun_out/kt257.json
timeout 300 python tools/kernel_table_at.py 513 > gpurun_out/kt513.json 2>>gpurun_out/kt.err; cat gpurun_out/kt513.json
timeout 900 python tools/run_config.py wedge3 --n 513 --maxit 4000 > gpurun_out/wedge513.json 2>gpurun_out/wedge.err; cat gpurun_out/wedge513.json
PROF_SOLVES=1 PROF_MAXIT=1 timeout 300 python tools/profile_solve.py > gpurun_out/plain.log 2>&1 && \
PROF_SOLVES=1 PROF_MAXIT=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'k_stencil|k_corr|k_restrict2|k_bcg' -c 14 -o gpurun_out/prof -f python tools/profile_solve.py > gpurun_out/ncu.log 2>&1
echo ncu exit $?; ls -la gpurun_out/
