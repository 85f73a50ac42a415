"""CPU: the C-ABI library builds/loads and exports every symbol that
include/wavepipe_b200.h declares (no compute calls without a GPU), and the
package has no CPU fallback path."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "wavepipe_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wp_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_seam():
    syms = declared_symbols()
    for name in ("wp_plan_create", "wp_plan_execute", "wp_iir_cascade", "wp_fir", "wp_white_noise", "wp_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2504_08624_b200 import _native
    from paper_2504_08624_b200._build import build_native

    path = build_native()
    lib = ctypes.CDLL(path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_native.EXPORTED) == declared_symbols()
    assert lib.wp_abi_version() == 1


def test_binary_is_sm100a_with_tensor_core_code():
    import shutil
    import subprocess

    from paper_2504_08624_b200._build import build_native

    path = build_native()
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", path], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out  # tcgen05.mma kind::f16
    assert "LDTM" in out     # tcgen05.ld


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2504_08624_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_no_gpu_means_loud_failure(monkeypatch):
    import numpy as np
    import torch

    import paper_2504_08624_b200 as wp

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    w = wp.Wave(np.ones((1, 32)), 44100) | wp.design_butterworth("lp", 2, 1000)
    with pytest.raises(wp.NativeUnavailable):
        w.samples
