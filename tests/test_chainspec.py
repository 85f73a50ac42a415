"""Chain-spec parser: every case of tests/golden/chainspec_golden.json (made
by the reference's own parser, make_chainspec_golden.py) - bound stages or
error class / column / message - is reproduced (chainspec.py:1-250)."""

import json
import os

import numpy as np
import pytest

import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import errors
from paper_2504_08624_b200.chainspec import FILTER_NAMES, parse_chain_spec

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "chainspec_golden.json")))


def test_catalog():
    assert FILTER_NAMES == ("butter", "cheby1", "fir", "hishelf", "loshelf", "peak")


@pytest.mark.parametrize("case", CASES, ids=[c["spec"][:40] or "<empty>" for c in CASES])
def test_chainspec_matches_reference(case):
    if "error" in case:
        with pytest.raises(errors.WavepipeError) as info:
            parse_chain_spec(case["spec"]).bind(48000)
        exc = info.value
        assert type(exc).__name__ == case["error"]
        assert getattr(exc, "column", None) == case["column"]
        assert str(exc) == case["message"]
        return
    bound = parse_chain_spec(case["spec"]).bind(48000).stages
    assert len(bound) == len(case["stages"])
    for st, ref in zip(bound, case["stages"]):
        if ref["type"] == "iir":
            assert isinstance(st, wp.IirFilter)
            assert st.overall_gain == pytest.approx(ref["gain"], rel=1e-12)
            got = np.array([[s.b0, s.b1, s.b2, s.a1, s.a2] for s in st.sections])
            np.testing.assert_allclose(got, np.array(ref["sections"]), rtol=1e-12, atol=1e-15)
        else:
            assert isinstance(st, wp.FirFilter)
            np.testing.assert_allclose(np.asarray(st.taps), np.array(ref["taps"]), rtol=1e-12, atol=1e-15)
