"""FIR strategy crossover on B200 (north_star: "tcgen05 Toeplitz GEMM or FFT
overlap-save, whichever is faster for the tap count, justified by ncu"): every tap count T runs
through each FIR kernel the planner can pick, on the same 32 x 2.88 M-sample workload:

  fir_tc   - tcgen05 f16x3 Hankel x Toeplitz GEMM    (strategy="direct", T within its smem range)
  fft_ols  - FFT overlap-save, 16 K complex points    (strategy="fft")
  cuda     - CUDA-core direct convolution (fused)     (WP_FIR_IMPL=cuda, T < 8 or as a reference)

python tools/fir_sweep.py            -> timing table (CUDA events, 10 passes after 3 warm-up)
python tools/fir_sweep.py --once     -> one pass per (T, kernel) for an ncu --metrics launch list
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import engine  # noqa: E402

TAPS = [8, 16, 32, 64, 101, 129, 192, 250, 257, 384, 512, 1024, 2048, 4096]
C, FS, DUR = 32, 48000, 60.0
N = int(FS * DUR)
once = "--once" in sys.argv
x = wp.white_noise(DUR, C, FS, seed=7).tensor()
y = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream
hbm = 6445.0
try:
    hbm = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass


def run(stages, strategy, env_cuda=False):
    if env_cuda:
        os.environ["WP_FIR_IMPL"] = "cuda"
    try:
        plan = engine.plan_for(stages, device=0, strategy=strategy)
    except Exception as e:  # strategy not available for this T
        return None, str(e).split("\n")[0][:60]
    finally:
        os.environ.pop("WP_FIR_IMPL", None)
    desc = plan.describe_for(C, N)[0]
    nb = plan.workspace_bytes(C, N)
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda")
    ex = lambda: plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)  # noqa: E731
    if once:
        ex()
        torch.cuda.synchronize()
        return 0.0, desc
    for _ in range(3):
        ex()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ex()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10, desc


rows = []
for T in TAPS:
    f = wp.design_fir("lp", T if T % 2 else T + 1, 15000).bind(FS)
    stages = wp.Chain([f]).bind(FS).stages
    res = {"T": len(f.taps)}
    for name, strat, envc in (("fir_tc", "direct", False), ("fft_ols", "fft", False), ("cuda", "direct", True)):
        if name == "cuda" and T > 512:
            continue  # the CUDA-core direct kernel is O(T) per sample: skip the long ones
        ms, desc = run(stages, strat, envc)
        kind = desc.split("[")[0].split(" ")[0] if ms is not None else None
        res[name] = {"ms": ms, "desc": desc, "kernel": kind}
    auto_ms, auto_desc = run(stages, "auto")
    res["auto"] = {"ms": auto_ms, "desc": auto_desc}
    rows.append(res)
    if not once:
        cells = []
        for name in ("fir_tc", "fft_ols", "cuda"):
            r = res.get(name)
            if not r or r["ms"] is None:
                cells.append("-")
            else:
                gcs = C * N / (r["ms"] * 1e-3) / 1e9
                cells.append(f"{r['ms']:.3f} ms ({gcs:.0f} G, {8 * gcs / hbm:.2f}) [{r['kernel']}]")
        print(f"T={res['T']:5d} | " + " | ".join(cells) + f" | auto -> {res['auto']['desc'].split(' ')[0]}", flush=True)
if not once:
    print(json.dumps(rows))
