#!/bin/bash
# GPU tests (all, or the files given in $TESTS) + a short configs[2] bench line (no CPU leg, no secondary solves)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -15 gpurun_out/t_gpu.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-tts > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/it", d["config"]["ms_per_iteration"], "clocks", d["clocks"])
for k, v in d["roofline"]["kernels"].items():
    print(f"  {k:20s} {v['ms']:8.4f} ms  {v['gbs']:8.1f} GB/s  frac {v['frac']:.3f}  share {v['share']}  bpv {v['bytes_per_vertex']}")
PY
tail -3 gpurun_out/bench_q.err
