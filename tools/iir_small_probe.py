"""IIR-only crossover: fused chunked scan vs chain_lb for small calls (LP4 = 2 SOS, LP8 = 4 SOS).
python tools/iir_small_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import _native, engine  # noqa: E402

fs = 48000
st = torch.cuda.current_stream().cuda_stream
for order in (4, 8):
    f = wp.design_butterworth("lp", order, 1000)
    bound = wp.Chain([f]).bind(fs).stages
    for C, N in ((1, 8192 * 4), (2, 8192 * 8), (2, 8192 * 16), (2, 441000), (4, 441000), (8, 441000), (16, 441000)):
        x = wp.white_noise(N / fs, C, fs, seed=1).tensor()
        y = torch.empty_like(x)
        res = []
        for impl in ("cuda", "lb"):
            os.environ["WP_CHAIN_IMPL"] = impl
            plan = _native.Plan(tuple(engine._entry(s) for s in bound))
            os.environ.pop("WP_CHAIN_IMPL")
            nb = plan.workspace_bytes(C, N)
            ws = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda")
            run = lambda: plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)  # noqa: E731
            for _ in range(5):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(50):
                run()
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / 50 * 1e3)
        tiles = C * -(-N // 8192)
        print(f"LP{order} C={C:3d} N={N:8d} tiles={tiles:5d}  fused {res[0]:7.1f} us  chain_lb {res[1]:7.1f} us")
