"""Generate tests/golden/cli_golden.json with the REFERENCE's CLI (build
container only: imports /root/reference/pkg/src): the exact text output of
``coeffs`` and ``response`` for a few chains, and exit codes of error cases."""

import json
import os
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
from wavepipe import cli  # noqa: E402

RUNS = [
    ["coeffs", "--chain", "butter(hp, 4, 100) | cheby1(lp, 4, 8000, 1.0) | fir(lp, 21, fc=15000)", "--fs", "48000"],
    ["coeffs", "--chain", "peak(1000, 3, q=2) | hishelf(fc=4000, gain_db=-6)", "--fs", "44100"],
    ["response", "--chain", "butter(lp, order=4, fc=1000) | hishelf(fc=1000, gain_db=3)", "--fs", "44100", "--points", "16"],
    ["response", "--chain", "fir(bp, 31, f1=500, f2=2000)", "--fs", "48000", "--points", "9"],
    ["coeffs", "--chain", "butter(lp 2)", "--fs", "48000"],
    ["coeffs", "--chain", "butter(lp, 2, 30000)", "--fs", "48000"],
    ["response", "--chain", "peak(1000, 3)", "--fs", "48000", "--points", "0"],
]


def main():
    out = []
    with tempfile.TemporaryDirectory() as d:
        for i, argv in enumerate(RUNS):
            path = os.path.join(d, f"o{i}.txt")
            code = cli.main(argv + ["--out", path])
            text = open(path).read() if os.path.exists(path) else None
            out.append({"argv": argv, "exit": code, "text": text})
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    for o in out:
        print(o["argv"][0], o["exit"], len(o["text"] or ""))


if __name__ == "__main__":
    main()
