#!/bin/bash
# evidence + large-config characterisation
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_evidence.sh k_flat_dr
for c in "wedge3 --n 513 --maxit 3000" "wedge3 --n 513 --method idrs --maxit 3000" "cube --n 257" "wedge3 --n 257"; do
  timeout 900 python tools/run_config.py $c >> gpurun_out/configs_final.jsonl 2>> gpurun_out/configs_final.err
done
cat gpurun_out/configs_final.jsonl | cut -c1-400
