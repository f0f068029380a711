#!/bin/bash
# round evidence for the bench workload (configs[2], 513^3 wedge):
#  * ncu --set full of one launch of every finest-level kernel on the default path
#    (tools/prof_wide2.py) -> DRAM traffic per kernel for bench.py, stall summary
#  * the launch list of two Bi-CGSTAB iterations (cold, serialised: compare shares)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PROF_PASSES=1 timeout -s KILL 300 python tools/prof_wide2.py > gpurun_out/pw4.log 2>&1 && \
PROF_PASSES=1 timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_wide|k_stencil|k_corr|k_restrict|k_bcg_p|k_bcg_s|k_bcg_xr" -c 10 \
  -o gpurun_out/wide4 -f python tools/prof_wide2.py > gpurun_out/ncu_wide4.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/ncu_wide4.log
export PROF_CONFIG=c2 PROF_SOLVES=1 PROF_MAXIT=4
timeout -s KILL 300 python tools/profile_solve.py > gpurun_out/plain.log 2>&1 && \
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python tools/profile_solve.py > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
