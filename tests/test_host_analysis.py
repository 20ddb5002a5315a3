"""Host-side analysis (paper_2404_11912_b200.host_analysis): the speedup
model against values computed by the reference itself
(tests/golden/make_golden_single.py), the Monte-Carlo model against the
closed form, and the planted-needle fixtures' invariants.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest


@pytest.fixture(scope="module")
def P():
    import paper_2404_11912_b200 as pkg
    return pkg


def test_expected_tokens(P):
    assert P.expected_tokens(0.0, 5) == 1.0
    assert P.expected_tokens(1.0, 4) == 5.0
    assert abs(P.expected_tokens(0.8, 4) - (1 - 0.8 ** 5) / 0.2) < 1e-12
    with pytest.raises(ValueError):
        P.expected_tokens(1.5, 2)
    with pytest.raises(ValueError):
        P.expected_tokens(0.5, -1)


def test_closed_form_speedup_matches_reference(P, golden_single):
    data, meta = golden_single
    for (a1, a2, g1, g2, ctx, b), want in zip(meta["speedup"]["grid"], data["speedup/values"]):
        r = P.hierarchical_speedup(a1, a2, g1, g2, P.LatencyModel(), ctx, b)
        c = P.hierarchical_speedup_coarse(a1, a2, g1, g2, P.LatencyModel(), ctx, b)
        got = [r.tokens_per_round, r.wall_ms_per_round, r.speedup, r.inner_rounds_per_outer,
               c.tokens_per_round, c.wall_ms_per_round, c.speedup, c.inner_rounds_per_outer]
        assert np.allclose(got, want, rtol=1e-12, atol=0), (a1, a2, g1, g2)


def test_monte_carlo_agrees_with_closed_form(P):
    lm = P.LatencyModel()
    for a1, a2, g1, g2 in ((0.8, 0.7, 2, 4), (0.5, 0.9, 3, 5), (0.95, 0.6, 1, 3)):
        exact = P.hierarchical_speedup(a1, a2, g1, g2, lm, 120000, 4096)
        mc = P.simulate_speedup(a1, a2, g1, g2, lm, 120000, 4096, rounds=20000, seed=3)
        assert abs(mc.speedup - exact.speedup) <= max(4 * mc.ci_halfwidth, 0.01 * exact.speedup), (a1, a2)
        assert abs(mc.inner_rounds_per_outer - exact.inner_rounds_per_outer) < 0.05 * exact.inner_rounds_per_outer
    with pytest.raises(ValueError):
        P.simulate_speedup(0.5, 0.5, 2, 4, lm, 1000, 100, rounds=10, seed=0)
    with pytest.raises(ValueError):   # full forward faster than the retrieval forward
        P.hierarchical_speedup(0.5, 0.5, 2, 4, P.LatencyModel(full_base=0.01, full_per_token=0.0), 1000, 100)


def test_needle_corpus_invariants(P):
    cases = P.needle_corpus(96, 20, seed=7)
    assert cases == P.needle_corpus(96, 20, seed=7)           # deterministic per seed
    for c in cases:
        assert len(c.tokens) == 96 and c.tokens[0] == P.BOS and c.tokens[-1] == ord("?")
        assert c.trigger_position == 95
        digits = [i for i, t in enumerate(c.tokens) if ord("0") <= t <= ord("9")]
        assert digits == c.needle_positions and len(digits) == 6
        assert bytes(c.tokens[i] for i in digits) == c.passkey
        assert int(np.ceil(0.1 * 96)) <= digits[0] and digits[-1] < int(np.floor(0.9 * 96))
    with pytest.raises(ValueError):
        P.needle_corpus(10, 1, seed=0)


def test_planted_attention_weights_construction(P):
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=8, d_ff=32, vocab_size=260, max_seq=512,
                        rope_theta=1e8)
    w = P.planted_attention_weights(cfg, 96, 6, strength=0.8, answer_token=ord("A"), seed=7)
    t = w.tensors
    d = cfg.d_model
    assert (t["embedding"][:, d - 2] == 1).all()
    assert (t["embedding"][list(range(48, 58)), d - 1] == 1).all() and t["embedding"][ord("a"), d - 1] == 0
    assert np.count_nonzero(t["lm_head"][d - 3]) == 1 and t["lm_head"][d - 3, ord("A")] == 1
    with pytest.raises(ValueError):
        P.planted_attention_weights(cfg, 96, 6, strength=1.0, answer_token=ord("A"))
    with pytest.raises(ValueError):
        P.planted_attention_weights(P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=8, d_ff=16,
                                                  vocab_size=260, max_seq=512), 96, 6, 0.8, ord("A"))


def test_monte_carlo_reproduces_reference_seeds(P):
    """Same draw order and batch means as the reference: a seed gives the
    reference's estimate (tests/golden/make_golden_mc.py)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "ref_mc.json")) as f:
        cases = json.load(f)
    for c in cases:
        a1, a2, g1, g2, ctx, b, rounds, seed = c["args"]
        r = P.simulate_speedup(a1, a2, g1, g2, P.LatencyModel(), ctx, b, rounds=rounds, seed=seed)
        got = [r.tokens_per_round, r.wall_ms_per_round, r.speedup, r.ci_halfwidth, r.inner_rounds_per_outer]
        assert np.allclose(got, c["result"], rtol=1e-12, atol=1e-12), c["args"]
