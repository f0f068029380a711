#!/bin/bash
# ncu --set full of the 513^3 wedge finest-level kernels the solve runs (one
# launch each, tools/prof_wide2.py) -> DRAM traffic per kernel for bench.py
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/prof_wide2.py > gpurun_out/pw2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stencil|k_corr|k_restrict|k_bcg" -c 8 \
  -o gpurun_out/wide3 -f python tools/prof_wide2.py > gpurun_out/ncu_wide3.log 2>&1
echo "ncu exit $?"
