#!/bin/bash
# wide-plane family: parity tests, then the A/B kernel table at 513^3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 420 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/t_wide.log 2>&1; tail -15 gpurun_out/t_wide.log
timeout -s KILL 200 python tools/ab_wide.py 513 > gpurun_out/ab_wide.log 2>&1; tail -5 gpurun_out/ab_wide.log
