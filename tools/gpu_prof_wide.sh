#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/prof_wide.py > gpurun_out/pw.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_down_restrict|k_stencil" -c 8 \
  -o gpurun_out/wide -f python tools/prof_wide.py > gpurun_out/ncu_wide.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_wide.log
