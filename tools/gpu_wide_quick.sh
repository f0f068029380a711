#!/bin/bash
# quick check of the wide-plane family: cycle parity subset, then A/B iteration times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_wide.py -x -q -k "cycle or solve" > gpurun_out/t_wide.log 2>&1; tail -4 gpurun_out/t_wide.log
timeout -s KILL 300 python tools/ab_iter.py ${AB_VARIANTS:-"" "no_wide_up=1"} > gpurun_out/ab_iter.log 2>&1; tail -5 gpurun_out/ab_iter.log
