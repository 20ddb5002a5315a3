"""TFWT weight files (reference weights_io.py) against a file written by the
reference's own writer (tests/golden/make_tfwt.py)."""

from __future__ import annotations

import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "tests", "golden", "ref_small.tfwt")


@pytest.fixture(scope="module")
def W():
    from paper_2404_11912_b200 import errors, model, weights_io
    return model, weights_io, errors


def _cfg(model):
    return model.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=8, d_ff=32, vocab_size=40, max_seq=128)


def test_load_reference_file_bitwise(W):
    model, wio, _ = W
    got = wio.load_weights(REF)
    want = model.generate_weights(_cfg(model), 11, tied_head=False)
    assert got.config == want.config and got.tied_head is False
    for name in want.tensors:
        assert np.array_equal(got.tensors[name].view(np.uint32), want.tensors[name].view(np.uint32)), name


def test_save_is_byte_identical_to_reference(W, tmp_path):
    model, wio, _ = W
    p = tmp_path / "w.tfwt"
    wio.save_weights(model.generate_weights(_cfg(model), 11, tied_head=False), p)
    assert p.read_bytes() == open(REF, "rb").read()
    t = tmp_path / "tied.tfwt"
    w = model.generate_weights(_cfg(model), 3, tied_head=True)
    wio.save_weights(w, t)
    back = wio.load_weights(t)
    assert back.tied_head and all(np.array_equal(back.tensors[k], w.tensors[k]) for k in w.tensors)


def test_format_errors(W, tmp_path):
    _, wio, err = W
    raw = open(REF, "rb").read()
    cases = [(b"XXXX" + raw[4:], err.BadMagicError), (raw[:4] + (2).to_bytes(4, "little") + raw[8:], err.VersionError),
             (raw[:-7], err.TruncatedFileError), (raw + b"\0", err.WeightFormatError),
             (raw[:8] + (0).to_bytes(4, "little") + raw[12:], err.WeightFormatError)]
    for i, (blob, exc) in enumerate(cases):
        p = tmp_path / f"bad{i}.tfwt"
        p.write_bytes(blob)
        with pytest.raises(exc):
            wio.load_weights(p)
    assert issubclass(err.BadMagicError, err.WeightFormatError)
