"""Shared fixtures. The ``gpu`` marker selects tests that need a B200; all other
tests run on CPU (oracle vs golden fixtures, host logic, ABI symbol export)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device and libwpb200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_vectors():
    return np.load(os.path.join(GOLDEN, "vectors.npz"))


@pytest.fixture(scope="session")
def golden_designs():
    with open(os.path.join(GOLDEN, "design.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_noise():
    with open(os.path.join(GOLDEN, "noise.json")) as fh:
        return json.load(fh)


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)


def sos_rows(entry):
    rows = np.array(entry["sections"], dtype=np.float64)
    rows[0, :3] *= entry["overall_gain"]
    return rows


def iir_from_entry(entry, fs):
    import paper_2504_08624_b200 as wp

    return wp.IirFilter.from_sections([tuple(r) for r in entry["sections"]], fs=fs, overall_gain=entry["overall_gain"])


def random_stable_section(rng):
    """conftest.random_stable_section of the reference (pkg/tests/conftest.py:29-42)."""
    import paper_2504_08624_b200 as wp

    if rng.random() < 0.7:
        radius = rng.uniform(0.0, 0.95)
        angle = rng.uniform(0.0, np.pi)
        a1, a2 = -2.0 * radius * np.cos(angle), radius * radius
    else:
        p1, p2 = rng.uniform(-0.95, 0.95, size=2)
        a1, a2 = -(p1 + p2), p1 * p2
    b = rng.uniform(-2.0, 2.0, size=3)
    return wp.BiquadSection(b[0], b[1], b[2], a1, a2)


def random_cascade(rng, max_sections=6, fs=44100):
    import paper_2504_08624_b200 as wp

    n = int(rng.integers(1, max_sections + 1))
    return wp.IirFilter.from_sections([random_stable_section(rng) for _ in range(n)], fs=fs,
                                      overall_gain=float(rng.uniform(0.25, 2.0)))


def random_unbound_stage(rng):
    """pkg/tests/conftest.py:52-64"""
    import paper_2504_08624_b200 as wp

    fc = float(rng.uniform(100, 8000))
    choice = int(rng.integers(0, 4))
    if choice == 0:
        kind = ("lowpass", "highpass")[int(rng.integers(0, 2))]
        return wp.design_butterworth(kind, int(rng.integers(1, 5)), fc)
    if choice == 1:
        return wp.design_chebyshev1("lowpass", int(rng.integers(1, 5)), float(rng.uniform(0.1, 2.0)), fc)
    if choice == 2:
        kind = ("lo_shelf", "hi_shelf")[int(rng.integers(0, 2))]
        return wp.design_shelf(kind, fc, gain_db=float(rng.uniform(-6, 6)))
    return wp.design_peaking(fc, gain_db=float(rng.uniform(-6, 6)), q=float(rng.uniform(0.5, 2.0)))
