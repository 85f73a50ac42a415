"""Run one config's plan a few times (for ncu launch lists / captures).
python tools/run_config.py cfg3 [reps]"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
import bench
import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import engine

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = bench.CONFIGS[name]
C, fs = cfg["C"], cfg["fs"]
dur = cfg["dur"] if name != "cfg5" else 20.0
N = int(round(dur * fs))
stages = wp.Chain(bench.stages_for(name, wp)).bind(fs).stages
x = wp.white_noise(dur, C, fs, seed=42).tensor()
y = torch.empty_like(x)
plan = engine.plan_for(stages, device=0)
print(plan.describe())
nb = plan.workspace_bytes(C, N)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
torch.cuda.synchronize()
