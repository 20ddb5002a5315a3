"""CPU-side checks of the boundary: the C-ABI library loads without a GPU and
exports every symbol `include/hs_abi.h` declares; host bookkeeping logic."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hs_abi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    b = __graft_entry__._builder()
    b.build()
    lib = ctypes.CDLL(b.LIB)
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.hs_abi_version() == 2


def test_python_binding_covers_the_header():
    from paper_2404_11912_b200 import _abi
    assert set(_declared()) <= set(_abi._SIGS)


def test_status_codes_map_to_reference_exceptions():
    from paper_2404_11912_b200 import _abi, errors
    for code, cls in ((-1, errors.ShapeError), (-2, errors.ContractError), (-3, errors.CapacityError),
                      (-4, errors.FiniteError)):
        try:
            _abi.check(code)
        except cls:
            pass
        else:
            raise AssertionError(code)


def test_streaming_watermark_matches_oracle_eviction():
    """Host-side StreamingCache bookkeeping (lo watermark) reproduces the
    oracle's physical eviction for random commit schedules."""
    from oracle import hs_oracle as O
    rng = np.random.default_rng(0)
    for trial in range(50):
        ns, budget = int(rng.integers(0, 4)), int(rng.integers(5, 20))
        W = budget - ns
        oc = O.OStreamingCache(1, 1, 2, ns, budget)
        lo, committed, frontier = ns, 0, 0
        for _ in range(30):
            t = int(rng.integers(1, 6))
            oc.append(0, np.zeros((t, 1, 2), np.float32), np.zeros((t, 1, 2), np.float32))
            frontier += t
            keep = int(rng.integers(0, t + 1))
            oc.rollback_to(committed + keep)
            frontier = committed + keep
            oc.commit(frontier)
            committed = frontier
            n_comm = min(committed, ns) + max(0, committed - max(lo, ns))
            if n_comm > budget:
                lo = max(lo, committed - W)
            store = np.concatenate([np.arange(min(ns, frontier)), np.arange(max(lo, ns), frontier)])
            assert store.tolist() == oc.rows[0].pos.tolist(), trial


def test_measure_acceptance_pairing_errors():
    """Pairing validation happens before any device work
    (analytics.py:296-300): unknown names raise ValueError."""
    import paper_2404_11912_b200 as P
    cfg = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=8, d_ff=16, vocab_size=16, max_seq=32)
    w = P.generate_weights(cfg, 1)
    with pytest.raises(ValueError):
        P.measure_acceptance("self:nope", w, [[1, 2, 3]])
    with pytest.raises(ValueError):
        P.measure_acceptance("hierarchical", w, [[1, 2, 3]])
    assert P.AcceptanceStats("x").rate == 0.0
