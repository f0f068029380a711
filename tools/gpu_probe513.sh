#!/bin/bash
# r02 probe: 513^3 wedge (configs[2]) kernel mix -- live kernel table and the
# ncu launch list of two Bi-CGSTAB iterations.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/kernel_table_at.py 513 wedge > gpurun_out/kt513w.json 2> gpurun_out/kt513w.err
timeout 600 python tools/run_config.py wedge3 --n 513 --maxit 40 > gpurun_out/w513_40.json 2> gpurun_out/w513_40.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_w513.csv python tools/run_config.py wedge3 --n 513 --maxit 2 \
  > gpurun_out/ncu_w513.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_w513.csv > gpurun_out/launches_w513_summary.txt 2>&1
