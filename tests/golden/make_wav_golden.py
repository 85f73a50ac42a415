"""Generate tests/golden/wav_golden.json with the REFERENCE's wavio (run in the
build container only: PYTHONPATH=/root/reference/pkg/src). Records, per
encoding, the sha256 of the file save_wav writes for a fixed float32-valued
signal (with samples beyond +-1 to exercise clipping), the clipped count, and
the sha256 of the samples load_wav reads back."""

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
from wavepipe import Wave, load_wav, save_wav  # noqa: E402


def signal():
    rng = np.random.default_rng(20261017)
    n = np.arange(4001)
    x = np.stack([1.3 * np.sin(2 * np.pi * 440 * n / 48000), 0.5 * rng.standard_normal(4001),
                  np.linspace(-1.0, 1.0, 4001)])
    x[2, ::7] = [0.5 / 32768, -0.5 / 32768, 1.5 / 32768, 2.5 / 8388608.0, -0.5 / 8388608.0, 1.0, -1.0][0]
    return x.astype(np.float32).astype(np.float64)


def main():
    x = signal()
    out = {"fs": 48000, "shape": list(x.shape), "signal_sha256": hashlib.sha256(x.tobytes()).hexdigest(), "cases": {}}
    with tempfile.TemporaryDirectory() as d:
        for enc in ("pcm16", "pcm24", "float32"):
            path = os.path.join(d, f"t_{enc}.wav")
            clipped = save_wav(Wave(x, 48000), path, encoding=enc)
            raw = open(path, "rb").read()
            back = load_wav(path)
            out["cases"][enc] = {"file_sha256": hashlib.sha256(raw).hexdigest(), "clipped": int(clipped),
                                 "decoded_sha256": hashlib.sha256(np.ascontiguousarray(back.samples).tobytes()).hexdigest(),
                                 "bytes": len(raw)}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "wav_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
