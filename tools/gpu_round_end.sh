#!/bin/bash
# round-end evidence: smoke(), bench line + launch list + ncu of the dominant
# kernel (tools/gpu_evidence.sh), and the 129^3 wedge kernel table and solve
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
bash tools/gpu_evidence.sh k_flat_dr
timeout 500 python tools/kernel_table_at.py 129 wedge > gpurun_out/ktw.json 2> gpurun_out/ktw.err
timeout 300 python tools/run_config.py wedge3 --n 129 > gpurun_out/w129.json 2>&1
echo done
