#!/bin/bash
# full check: every GPU test, smoke(), the default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu_full.log 2>&1; tail -5 gpurun_out/t_gpu_full.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
