"""Diagnostics: time IIR-only passes (cfg3's IIR part, cfg5 slice, cfg1) on
the current kernel selection (WP_CHAIN_IMPL=cuda forces the CUDA-core kernel)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import engine

def run(label, stages, C, fs, dur, reps=10):
    N = int(dur * fs)
    w = wp.white_noise(dur, C, fs, seed=42); x = w.tensor(); y = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    plan = engine.plan_for(wp.Chain(stages).bind(fs).stages, device=0)
    nb = plan.workspace_bytes(C, N); ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for _ in range(3): plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{label:28s} {ms:8.3f} ms  {C*N/ms/1e6:8.1f} G ch-s/s  {plan.describe()[0][:60]}")

run("cfg3 IIR (HP4|Cheb4) f64", [wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000)], 32, 48000, 120.0)
run("cfg5 LP8 (100 s slice)", [wp.design_butterworth("lp", 8, 2000)], 1024, 48000, 20.0)
run("cfg1 LP4", [wp.design_butterworth("lp", 4, 1000)], 2, 44100, 10.0, reps=50)
run("cfg3 full chain", [wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000), wp.design_fir("lp", 101, 15000), wp.Gain(0.5)], 32, 48000, 120.0)
