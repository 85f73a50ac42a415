"""Run one config's fused plan a few times (for ncu captures): python tools/run_plan.py cfg3 [seconds] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = bench.CONFIGS[name]
C, fs = cfg["C"], cfg["fs"]
dur = float(sys.argv[2]) if len(sys.argv) > 2 else cfg["dur"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
N = int(round(dur * fs))
stages = wp.Chain(bench.stages_for(name, wp)).bind(fs).stages
x = wp.white_noise(dur, C, fs, seed=42).tensor()
y = torch.empty_like(x)
plan = engine.plan_for(stages, device=0)
print(plan.describe_for(C, N))
nb = plan.workspace_bytes(C, N)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
torch.cuda.synchronize()
