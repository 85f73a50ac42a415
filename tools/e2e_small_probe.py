"""e2e (pinned host -> device -> host through the public API) of cfg1-cfg3 with
the streamed host path cut into different channel-block counts, same box:
python tools/e2e_small_probe.py [reps]"""
import statistics
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__file__), ".."))
import bench  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import engine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for name in ("cfg1", "cfg2", "cfg3"):
    cfg = bench.CONFIGS[name]
    C, fs = cfg["C"], cfg["fs"]
    N = int(round(cfg["dur"] * fs))
    host_in = torch.randn((C, N), dtype=torch.float32).pin_memory()
    host_out = torch.empty((C, N), dtype=torch.float32, pin_memory=True)
    chain = wp.Chain(bench.stages_for(name, wp))
    entries = (wp.Wave.from_tensor(host_in, fs) | chain)._entries
    for blocks in sorted({max(1, (C + 1) // 2), C, min(C, 16)}):
        def step():
            engine.stream_host_entries(entries, host_in, host_out, blocks=blocks)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            step()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(f"{name} C={C} blocks={blocks}: median {statistics.median(ts)*1e3:.3f} ms  "
              f"min {min(ts)*1e3:.3f} ms  -> {C*N/statistics.median(ts)/1e9:.2f} G ch-s/s", flush=True)
    # the full public call (design cache, lazy pipe, numpy32) at the default block rule
    def api():
        (wp.Wave.from_tensor(host_in, fs) | chain).numpy32(out=host_out)
    for _ in range(3):
        api()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        api()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name} public API: median {statistics.median(ts)*1e3:.3f} ms -> {C*N/statistics.median(ts)/1e9:.2f} G ch-s/s",
          flush=True)
