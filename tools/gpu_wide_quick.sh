#!/bin/bash
# quick check: cycle / solve parity subsets, kernel table, iteration time
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "cycle or solve or bicgstab or shadow or configs" > gpurun_out/t_wide.log 2>&1; tail -4 gpurun_out/t_wide.log
timeout -s KILL 300 python tools/kernel_table_at.py 513 wedge > gpurun_out/kt.json 2>gpurun_out/kt.err; tail -c 300 gpurun_out/kt.err
timeout -s KILL 300 python tools/ab_iter.py ${AB_VARIANTS:-""} > gpurun_out/ab_iter.log 2>&1; tail -5 gpurun_out/ab_iter.log
