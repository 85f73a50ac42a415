"""WAV codec: the oracle restatement is pinned to the reference's own save_wav /
load_wav output (tests/golden/wav_golden.json, made by make_wav_golden.py
from /root/reference), and the device codec reproduces it byte for byte."""

import hashlib
import json
import os
import struct

import numpy as np
import pytest

import oracle
import paper_2504_08624_b200 as wp

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "wav_golden.json")))


def signal():
    # identical to tests/golden/make_wav_golden.py
    rng = np.random.default_rng(20261017)
    n = np.arange(4001)
    x = np.stack([1.3 * np.sin(2 * np.pi * 440 * n / 48000), 0.5 * rng.standard_normal(4001),
                  np.linspace(-1.0, 1.0, 4001)])
    x[2, ::7] = [0.5 / 32768, -0.5 / 32768, 1.5 / 32768, 2.5 / 8388608.0, -0.5 / 8388608.0, 1.0, -1.0][0]
    return x.astype(np.float32).astype(np.float64)


def sha(b):
    return hashlib.sha256(b).hexdigest()


def test_signal_is_the_golden_one():
    assert sha(signal().tobytes()) == GOLDEN["signal_sha256"]


@pytest.mark.parametrize("enc", ["pcm16", "pcm24", "float32"])
def test_oracle_codec_pinned_to_reference(enc):
    case = GOLDEN["cases"][enc]
    raw, clipped = oracle.wav_file_bytes(signal(), GOLDEN["fs"], enc)
    assert sha(raw) == case["file_sha256"] and len(raw) == case["bytes"]
    assert clipped == case["clipped"]
    payload_len = struct.unpack_from("<I", raw, 40)[0]
    back = oracle.wav_decode(raw[44:44 + payload_len], enc, 3)
    assert sha(np.ascontiguousarray(back).tobytes()) == case["decoded_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("enc", ["pcm16", "pcm24", "float32"])
def test_device_codec_byte_exact(enc, tmp_path):
    case = GOLDEN["cases"][enc]
    path = tmp_path / f"dev_{enc}.wav"
    clipped = wp.save_wav(wp.Wave(signal(), GOLDEN["fs"]), path, encoding=enc)
    assert sha(path.read_bytes()) == case["file_sha256"]
    assert clipped == case["clipped"]
    back = wp.load_wav(path)
    assert back.fs == GOLDEN["fs"] and back.shape == tuple(GOLDEN["shape"])
    assert sha(np.ascontiguousarray(back.samples).tobytes()) == case["decoded_sha256"]


@pytest.mark.gpu
def test_device_codec_large_multichannel_roundtrip(tmp_path):
    w = wp.white_noise(2.0, 37, 48000, seed=4)  # many channels, odd count, device-generated
    path = tmp_path / "big.wav"
    wp.save_wav(w, path, encoding="float32")
    assert wp.load_wav(path) == w
    ref, _ = oracle.wav_file_bytes(w.samples, 48000, "pcm24")
    wp.save_wav(w, tmp_path / "p24.wav", encoding="pcm24")
    assert (tmp_path / "p24.wav").read_bytes() == ref


@pytest.mark.gpu
def test_device_codec_errors(tmp_path):
    bad = tmp_path / "bad.wav"
    bad.write_bytes(b"RIFF\x04\x00\x00\x00WAVE")
    with pytest.raises(wp.MalformedRiff):
        wp.load_wav(bad)
    raw, _ = oracle.wav_file_bytes(signal(), 48000, "pcm16")
    alaw = bytearray(raw)
    struct.pack_into("<H", alaw, 20, 6)  # format tag 6 (A-law)
    (tmp_path / "alaw.wav").write_bytes(bytes(alaw))
    with pytest.raises(wp.UnsupportedEncoding):
        wp.load_wav(tmp_path / "alaw.wav")
    with pytest.raises(wp.UnsupportedEncoding):
        wp.save_wav(wp.Wave(signal(), 48000), tmp_path / "x.wav", encoding="pcm8")


@pytest.mark.gpu
@pytest.mark.parametrize("enc", ["pcm16", "pcm24", "float32"])
@pytest.mark.parametrize("chunk_bytes", [1000, 64 << 10])
def test_chunked_stream_matches_single_chunk(enc, chunk_bytes, tmp_path):
    """The double-buffered chunked file <-> device pipeline (many chunks, a last
    partial chunk, frames not aligned to anything) writes the same bytes as the
    reference's writer and reads back the same values."""
    w = wp.white_noise(0.7, 5, 44100, seed=9)  # 30870 frames x 5 ch
    path = tmp_path / f"c_{enc}.wav"
    clipped = wp.save_wav(w, path, encoding=enc, chunk_bytes=chunk_bytes)
    ref, ref_clipped = oracle.wav_file_bytes(w.samples, 44100, enc)
    assert path.read_bytes() == ref
    assert clipped == (ref_clipped if enc != "float32" else 0)
    one = wp.load_wav(path)  # one chunk
    many = wp.load_wav(path, chunk_bytes=chunk_bytes)
    assert np.array_equal(one.samples, many.samples)
    if enc == "float32":
        assert many == w
