#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/prof_wide2.py > gpurun_out/pw2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stencil|k_corr|k_restrict|k_bcg" -c 12 \
  -o gpurun_out/wide2 -f python tools/prof_wide2.py > gpurun_out/ncu_wide2.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_wide2.log
