"""Time one V-cycle (mg_precondition on device tensors) of the 129^3 CSLP
hierarchy while the k_coarse phase list is truncated to HF_COARSE_NPH phases
(timing only: truncated cycles are wrong), and with k_coarse off (the default; HF_COARSE=1 turns it on)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, mg_precondition
from paper_2308_06085_b200.operators import OperatorSpec
p, spec, b = bench._problem()
H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
r = torch.as_tensor(b).cuda(); z = torch.empty_like(r)
for _ in range(5): mg_precondition(H, r, out=z)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50): mg_precondition(H, r, out=z)
e.record(); torch.cuda.synchronize()
print(round(s.elapsed_time(e) / 50 * 1e3, 2))
'''

def run(env):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True)
    return out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]

print("no k_coarse:", run({}), "us/cycle")
for n in range(0, 12):
    print(f"nph={n}:", run({"HF_COARSE": "1", "HF_COARSE_NPH": str(n)}), "us/cycle")
for n in (1, 2, 6, 11):
    print(f"nph={n} barriers only:", run({"HF_COARSE": "1", "HF_COARSE_NPH": str(n), "HF_COARSE_NOP": "1"}), "us/cycle")
