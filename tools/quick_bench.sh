# GPU check used while iterating: gpu tests, then two short bench runs summarised
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print(d['ms_per_step'], d['config']['iterations'], round(d['ms_per_step']/d['config']['iterations']*1e3,1), 'us/it', {a:b['ms'] for a,b in k.items()})"
done
