#!/bin/bash
# quick GPU check: gpu tests (unless NO_TESTS=1), then A/B bench lines (summarised)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/quick.txt
if [ -z "$NO_TESTS" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -1 gpurun_out/t_gpu.log | tee -a gpurun_out/quick.txt
fi
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print(d['ms_per_step'], d['config']['iterations'], round(d['ms_per_step']/d['config']['iterations']*1e3,1), 'us/it', 'e2e', d['e2e']['ms_per_step'], {a:b['ms'] for a,b in k.items()})"; }
for v in "$@"; do
  echo "== $v" | tee -a gpurun_out/quick.txt
  env $v timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 2>gpurun_out/bench_err.log | summ | tee -a gpurun_out/quick.txt
done
