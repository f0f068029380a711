#!/bin/bash
# wide-plane family: parity tests, then the strip-height A/B at 513^3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/t_wide.log 2>&1; tail -5 gpurun_out/t_wide.log
timeout -s KILL 300 python tools/ab_iter.py "" "wide_p3=1" "wide_p4=1" > gpurun_out/ab_iter.log 2>&1; tail -4 gpurun_out/ab_iter.log
