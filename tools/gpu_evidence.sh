#!/bin/bash
# round evidence for the bench workload (configs[2], 513^3 wedge): the launch
# list of two Bi-CGSTAB iterations (cold, serialised: compare shares) and one
# ncu --set full capture of the dominant kernel, summarised into profiles/
#   bash tools/gpu_evidence.sh <kernel regex> [bench kernel name]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PROF_CONFIG=c2 PROF_SOLVES=1 PROF_MAXIT=2 timeout 300 python tools/profile_solve.py > gpurun_out/plain.log 2>&1 && \
  PROF_CONFIG=c2 PROF_SOLVES=1 PROF_MAXIT=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python tools/profile_solve.py > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
PROF_CONFIG=c2 PROF_SOLVES=1 PROF_MAXIT=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"$1" -c 1 -o gpurun_out/dom_c2 -f python tools/profile_solve.py > gpurun_out/ncu_dom.log 2>&1
echo "ncu dom exit $?"
