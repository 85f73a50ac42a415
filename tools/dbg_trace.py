import sys, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import bench, paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import _native, engine
cfg = bench.CONFIGS['cfg3']; C, fs = cfg['C'], cfg['fs']; dur = 1.0; N = int(dur*fs)
stages = wp.Chain(bench.stages_for('cfg3', wp)).bind(fs).stages
w = wp.white_noise(dur, C, fs, seed=42); x = w.tensor(); y = torch.empty_like(x)
plan = engine.plan_for(stages, device=0); print(plan.describe())
nb = plan.workspace_bytes(C, N); ws = torch.empty(nb, dtype=torch.uint8, device='cuda')
st = torch.cuda.current_stream().cuda_stream
tiles = C * ((N + 8191)//8192); tr = torch.zeros(tiles*12, dtype=torch.int64, device='cuda')
_native.set_trace(tr.data_ptr(), tr.numel())
plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
torch.cuda.synchronize()
print('trace nonzero', int((tr != 0).sum()), 'of', tr.numel())
print('y finite', bool(torch.isfinite(y).all()), float(y.abs().max()))
