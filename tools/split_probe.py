"""Diagnostics: time the cfg3 chain's IIR part and FIR part as separate passes
(CUDA-core fused IIR kernel vs tensor-core chain; fir_tc for the FIR)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import engine

fs, C, dur = 48000, 32, 120.0
N = int(dur * fs)
w = wp.white_noise(dur, C, fs, seed=42)
x = w.tensor(); y = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream
def timeit(stages, label):
    plan = engine.plan_for(wp.Chain(stages).bind(fs).stages, device=0)
    nb = plan.workspace_bytes(C, N); ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for _ in range(3): plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
    e1.record(); torch.cuda.synchronize()
    print(f"{label:40s} {e0.elapsed_time(e1)/10:.3f} ms  {plan.describe()}")
iir = [wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000)]
fir = [wp.design_fir("lp", 101, 15000), wp.Gain(0.5)]
timeit(iir, "IIR (HP4|Cheb4) " + os.environ.get("WP_CHAIN_IMPL", "tc"))
timeit(fir, "FIR101 + gain")
timeit(iir + fir, "full chain " + os.environ.get("WP_CHAIN_IMPL", "tc"))
