"""The CPU baseline's fidelity: the oracle port (oracle/wp_oracle.c, the
`cpu_baseline` / `--impl reference` arm on the GPU box) against the UNMODIFIED reference
(`wavepipe` with numba, imported read-only from /root/reference) on the same host, same
data, same thread count, for every BASELINE config's stage list on a time slice.

Runs in the development container only (the reference cannot travel to the GPU box):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/port_vs_numba.py > profiles/r2_port_vs_numba.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import oracle  # noqa: E402
import wavepipe as ref  # noqa: E402
from wavepipe import engine as ref_engine  # noqa: E402

threads = os.cpu_count() or 1
ref_engine.set_num_threads(threads)


def ref_stages(name):
    if name == "cfg1":
        return [ref.design_butterworth("lowpass", 4, 1000.0)]
    if name == "cfg2":
        return [ref.design_fir("lowpass", 101, 1000.0, "hamming")]
    if name == "cfg3":
        return [ref.design_butterworth("highpass", 4, 100.0), ref.design_chebyshev1("lowpass", 4, 1.0, 8000.0),
                ref.design_fir("lowpass", 101, 15000.0)]
    if name == "cfg4":
        return [ref.design_fir("lowpass", 4096, 2000.0, "hamming")]
    if name == "cfg5":
        return [ref.design_butterworth("lowpass", 8, 2000.0)]


cfgs = {"cfg1": (2, 44100, 10.0), "cfg2": (8, 48000, 6.0), "cfg3": (32, 48000, 2.0), "cfg4": (128, 48000, 0.5),
        "cfg5": (64, 48000, 2.0)}
out = {"threads": threads, "host": os.uname().nodename, "configs": {}}
for name, (C, fs, dur) in cfgs.items():
    x = oracle.white_noise(dur, C, fs, 42).astype(np.float32).astype(np.float64)
    stages = [s.bind(fs) for s in ref_stages(name)]
    w = ref.Wave(x, fs)

    def run_ref():
        y = w
        for s in stages:
            y = s.apply(y)
        return y.samples

    def run_port():
        return oracle.pipe(x, stages, threads)

    for f in (run_ref, run_port):
        f()  # warm-up (numba JIT / oracle library)
    res = {}
    for label, f in (("reference_numba", run_ref), ("oracle_port", run_port)):
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            y = f()
            ts.append(time.perf_counter() - t0)
        res[label] = {"s": min(ts), "ch_samples_per_s": C * x.shape[1] / min(ts)}
    a, b = run_ref(), run_port()
    res["max_abs_diff"] = float(np.max(np.abs(a - b)))
    res["port_over_reference"] = res["oracle_port"]["ch_samples_per_s"] / res["reference_numba"]["ch_samples_per_s"]
    res["slice"] = f"{C} ch x {x.shape[1]} frames"
    out["configs"][name] = res
    print(name, json.dumps(res), file=sys.stderr)
print(json.dumps(out, indent=1))
