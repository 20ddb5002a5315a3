"""Shared test setup.

`-m gpu` tests need a B200 and the in-tree CUDA library; everything else runs
on CPU.  The oracle (`oracle/hs_oracle.py`) is test infrastructure and is
imported here only as the checker.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN_DIR, "ref_golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "ref_golden.json")) as f:
        meta = json.load(f)
    return data, meta


@pytest.fixture(scope="session")
def golden_single():
    """One-level speculation fixtures (tests/golden/make_golden_single.py)."""
    data = np.load(os.path.join(GOLDEN_DIR, "ref_single.npz"))
    with open(os.path.join(GOLDEN_DIR, "ref_single.json")) as f:
        meta = json.load(f)
    return data, meta


def small_cfg(**kw):
    from oracle.hs_oracle import OConfig
    base = dict(n_layers=2, n_heads=4, n_kv_heads=4, head_dim=8, d_ff=32,
                vocab_size=40, max_seq=128, rope_theta=10000.0, norm_eps=1e-5)
    base.update(kw)
    return OConfig(**base)
