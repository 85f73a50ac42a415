"""File -> GPU chain -> file throughput: a cfg3-shaped WAV (32 ch x 48 kHz x
120 s float32, 737 MB) through load_wav | HP4 | Cheb LP4 | FIR 101 | gain | save_wav, with the
chunked double-buffered pipeline (64 MiB chunks) and with one chunk (the round-1 behaviour),
plus the host-only numpy decode of the same file (what the reference's wavio.load_wav does).

python tools/wav_stream_bench.py [seconds]      (files under /tmp; the page cache holds them)
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2504_08624_b200 as wp  # noqa: E402

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
C, FS = 32, 48000
src, dst = "/tmp/wpb_in.wav", "/tmp/wpb_out.wav"
w = wp.white_noise(dur, C, FS, seed=42)
wp.save_wav(w, src, encoding="float32")
size = os.path.getsize(src)
chain = (wp.design_butterworth("hp", 4, 100) | wp.design_chebyshev1("lp", 4, 1.0, 8000)
         | wp.design_fir("lp", 101, 15000) | wp.Gain(0.5))


def run(chunk):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = wp.load_wav(src, chunk_bytes=chunk)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    y = x | chain
    yt = y.tensor()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    wp.save_wav(y, dst, encoding="float32", chunk_bytes=chunk)
    t3 = time.perf_counter()
    del yt
    return t1 - t0, t2 - t1, t3 - t2, t3 - t0


res = {}
for name, chunk in (("chunked_32MiB_x4", 32 << 20), ("one_chunk", 1 << 40)):
    run(chunk)  # warm-up (page cache, pinned allocator, plan cache)
    best = min((run(chunk) for _ in range(3)), key=lambda r: r[3])
    res[name] = {"load_s": best[0], "chain_s": best[1], "save_s": best[2], "total_s": best[3],
                 "file_to_file_GBps": 2 * size / best[3] / 1e9,
                 "ch_samples_per_s": C * dur * FS / best[3]}
# host-only decode of the same file with numpy (the reference's wavio.load_wav path)
t0 = time.perf_counter()
raw = np.fromfile(src, dtype=np.uint8)
data = raw[44:].view("<f4").reshape(-1, C).T.astype(np.float64)
res["numpy_decode_only_s"] = time.perf_counter() - t0
res["file_bytes"] = size
print(json.dumps(res, indent=1))
