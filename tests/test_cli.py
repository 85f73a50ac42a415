"""CLI: ``coeffs`` / ``response`` text and exit codes identical to the
reference's CLI (tests/golden/cli_golden.json, make_cli_golden.py); on a GPU,
``noise`` + ``apply`` run end to end through the device WAV codec and one
fused plan, matching the oracle within the chain tolerance."""

import json
import os

import numpy as np
import pytest

import oracle
from paper_2504_08624_b200 import cli

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cli_golden.json")))


@pytest.mark.parametrize("case", CASES, ids=[" ".join(c["argv"][:3])[:50] for c in CASES])
def test_cli_text_and_exit_codes_match_reference(case, tmp_path):
    out = tmp_path / "o.txt"
    code = cli.main(case["argv"] + ["--out", str(out)])
    assert code == case["exit"]
    if case["text"] is None:
        assert not out.exists()
    else:
        assert out.read_text() == case["text"]


def test_cli_missing_input_is_io_error(tmp_path):
    assert cli.main(["apply", str(tmp_path / "nope.wav"), str(tmp_path / "o.wav"), "--chain", "peak(1000, 3)"]) in (
        cli.EXIT_IO, cli.EXIT_FILTER)


@pytest.mark.gpu
def test_cli_noise_apply_end_to_end(tmp_path):
    src, dst = tmp_path / "n.wav", tmp_path / "y.wav"
    assert cli.main(["noise", "--duration", "2", "--channels", "2", "--fs", "44100", "--seed", "20260809",
                     "--out", str(src)]) == 0
    spec = "butter(lp, order=4, fc=1000) | hishelf(fc=1000, gain_db=3) | fir(lp, 31, fc=5000)"
    assert cli.main(["apply", str(src), str(dst), "--chain", spec]) == 0
    x, fs = oracle.load_wav_float32(str(src))
    y, fs2 = oracle.load_wav_float32(str(dst))
    assert fs == fs2 == 44100
    from paper_2504_08624_b200.chainspec import parse_chain_spec

    ref = oracle.pipe(x, parse_chain_spec(spec).bind(44100).stages)
    assert oracle.parity_error(y, ref) <= 1e-4
    # the input noise is the reference generator's stream (float32-rounded)
    assert np.max(np.abs(x - oracle.white_noise(2.0, 2, 44100, 20260809))) <= 1e-6
