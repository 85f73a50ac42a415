"""Generate tests/golden/chainspec_golden.json with the REFERENCE's chain-spec
parser (build container only: imports /root/reference/pkg/src). Each case
records either the bound stages (fs = 48000: sections / taps) or the error
(class, column, message)."""

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
from wavepipe import errors  # noqa: E402
from wavepipe.chainspec import parse_chain_spec  # noqa: E402

SPECS = [
    "butter(lp, order=4, fc=1000) | hishelf(fc=1000, gain_db=3)",
    "hishelf(fc=1000, gain_db=3) | loshelf(fc=2000, gain_db=3)",
    "butter(lp, order=4, fc=1000)",
    "peak(fc=1000,gain_db=2)|peak(fc=2000,gain_db=-2)",
    "  peak( fc = 1000 , gain_db = 2 )  |  peak( fc = 2000 , gain_db = -2 )  ",
    "peak(1000, 3, q=2)",
    "fir(lp, num_taps=31, fc=2000, window=blackman) | fir(bp, 31, f1=500, f2=2000)",
    "cheby1(lp, order=4, fc=2e3, ripple_db=1e0)",
    "butter(hp, 4, 100) | cheby1(lp, 4, 8000, 1.0) | fir(lp, 101, fc=15000)",
    "butter(lp, order=0, fc=100)",
    "peak(fc=1000, gain_db=1) | warble(fc=2)",
    "peak(fc=1000, gain_db=1, slope=2)",
    "hishelf(fc=1000)",
    "fir(bp, num_taps=31)",
    "fir(lp, 31)",
    "peak(fc=1000 gain_db=1)",
    "peak fc=1000",
    "",
    "peak(fc=1000, gain_db=1) peak(fc=2, gain_db=1)",
    "peak(fc=1000, gain_db=1) @ peak(fc=1, gain_db=1)",
    "peak(1000, fc=2000, gain_db=1)",
    "peak(fc=1000, 3)",
    "peak(1000, 3, 1, 7)",
    "peak(fc=1000, fc=2000, gain_db=1)",
    "butter(lp, 4, 30000)",
    "peak(fc=1e3, gain_db=-.5, q=.7)",
    "fir(hp, 32, fc=1000)",
    "butter(",
    "butter(lp, 4, 100",
]


def stage_json(st):
    if hasattr(st, "sections"):
        return {"type": "iir", "gain": st.overall_gain,
                "sections": [[s.b0, s.b1, s.b2, s.a1, s.a2] for s in st.sections]}
    return {"type": "fir", "taps": [float(t) for t in st.taps]}


def main():
    cases = []
    for spec in SPECS:
        try:
            chain = parse_chain_spec(spec)
            bound = chain.bind(48000)
            cases.append({"spec": spec, "stages": [stage_json(s) for s in bound.stages]})
        except errors.WavepipeError as exc:
            cases.append({"spec": spec, "error": type(exc).__name__, "column": getattr(exc, "column", None),
                          "message": str(exc)})
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "chainspec_golden.json")
    with open(out, "w") as fh:
        json.dump(cases, fh, indent=1)
    for c in cases:
        print(c["spec"][:50], "->", c.get("error", len(c.get("stages", []))), c.get("column", ""))


if __name__ == "__main__":
    main()
