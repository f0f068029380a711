#!/bin/bash
# ncu --set full of the wide-plane family (k_wide) on the 513^3 wedge finest level
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export HF_PROF_OPTS="${HF_PROF_OPTS:-}"
timeout -s KILL 200 python tools/prof_wide2.py > gpurun_out/pw3.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_wide" -c 3 \
  -o gpurun_out/wide_kw -f python tools/prof_wide2.py > gpurun_out/ncu_wide_kw.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_wide_kw.log
