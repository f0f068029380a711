#!/bin/bash
# A/B of a k_flat_dr change: parity tests on the new build, then alternating
# bench lines against the previous build (paper_2308_06085_b200/_lib/libhelmfree_b200_old.so)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -x -q > gpurun_out/t_ab.log 2>&1; tail -1 gpurun_out/t_ab.log > gpurun_out/ab.txt
OLD=HF_LIB_PATH=$PWD/paper_2308_06085_b200/_lib/libhelmfree_b200_old.so
NO_TESTS=1 bash tools/gpu_quick.sh "$OLD" "HF_X=0" "$OLD" "HF_X=0" "$@"
cat gpurun_out/quick.txt >> gpurun_out/ab.txt
