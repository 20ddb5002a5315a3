"""One-level speculation on the B200 (`-m gpu`): `SingleLevelSession`
(speculation.py:401-477) and `measure_acceptance` (analytics.py:265-309)
against fixtures produced by the reference itself
(tests/golden/make_golden_single.py, bf16 storage model), plus the
reference's own properties (tests/test_speculation.py:336-362,
tests/test_acceptance.py:144-162)."""

from __future__ import annotations

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2404_11912_b200 as pkg
    return pkg


def bf16_weights(P, w):
    from oracle.hs_oracle import bf16_round
    t = {n: (x.copy() if "norm" in n else bf16_round(x)) for n, x in w.tensors.items()}
    return P.ModelWeights(w.config, t, w.tied_head).validate()


@pytest.fixture(scope="module")
def needle(P, golden_single):
    data, meta = golden_single
    target = bf16_weights(P, P.load_weights(os.path.join(HERE, "golden", "needle.tfwt")))
    cfg = dict(target.config.__dict__)
    cfg["n_layers"] = 1
    draft = bf16_weights(P, P.generate_weights(P.ModelConfig(**cfg), meta["single_sessions"]["draft_seed"]))
    prompts = [list(map(int, p)) for p in data["needle/prompts"]]
    return target, draft, prompts


def _draft_cache(P, kind, cfg, kw):
    if kind == "full":
        return P.FullCache.from_config(cfg)
    if kind == "topk":
        return P.TopKCache.from_config(cfg, kw["budget"])
    if kind == "h2o":
        return P.H2OCache.from_config(cfg, P.H2OConfig(**kw))
    if kind == "stream":
        return P.StreamingCache.from_config(cfg, P.StreamingConfig(**kw))
    return P.RetrievalCache.from_config(cfg, P.RetrievalConfig(**kw))


def test_single_level_sessions_match_reference(P, golden_single, needle):
    data, meta = golden_single
    target, draft, prompts = needle
    for c in meta["single_sessions"]["cases"]:
        dw = target if c["self_spec"] else draft
        cache = _draft_cache(P, c["kind"], dw.config, c["cache"])
        prefix = prompts[c["prompt_case"]]
        s = P.SingleLevelSession(dw, cache, target, prefix, c["gamma"], c["temperature"])
        out, st = s.generate(len(prefix) + c["gen"], seed=c["seed"])
        tag = f"single/{c['name']}/bf16"
        assert out == data[tag + "/tokens"].tolist(), c["name"]
        assert [st.rounds, st.proposed, st.accepted] == data[tag + "/stats"].tolist(), c["name"]
        if c["kind"] == "h2o":   # the surviving entries (exact) and their heavy-hitter scores (the
            # probabilities come from our forward's fp32 q, so they agree to ~1e-6 relative), per layer
            for li in range(dw.config.n_layers):
                assert cache.exposed_positions(li).tolist() == data[tag + f"/exposed{li}"].tolist(), (c["name"], li)
                sc = cache.cumulative_scores(li)
                got = np.array([sc[p] for p in sorted(sc)])
                assert np.allclose(got, data[tag + f"/scores{li}"], rtol=1e-5, atol=1e-9), (c["name"], li)


def test_needle_acceptance_matches_reference_and_orders_pairings(P, golden_single, needle):
    """Acceptance criterion 3 on the device path: top-k exposure (the oracle
    upper bound) >= retrieval drafting > streaming, with an alpha gap >= 0.3
    between retrieval and streaming, and every case's counts equal the
    reference's."""
    data, meta = golden_single
    target, _, prompts = needle
    m = meta["needle"]
    kw = dict(gamma=m["gamma"], temperature=m["temperature"], gen_tokens=m["gen_tokens"], seed=m["seed"],
              streaming=P.StreamingConfig(n_sink=m["n_sink"], budget=m["budget"]),
              retrieval=P.RetrievalConfig(chunk_size=m["chunk_size"], budget=m["budget"]), topk_budget=m["budget"],
              h2o=P.H2OConfig(budget=m["budget"], recent_window=m["h2o_recent_window"]))
    rates = {}
    for kind in ("retrieval", "streaming", "topk", "h2o"):
        st = P.measure_acceptance("self:" + kind, target, prompts, **kw)["self"]
        tag = f"needle/bf16/{kind}"
        assert [st.rounds, st.proposed, st.accepted] == data[tag + "/stats"].tolist(), kind
        assert np.array_equal(np.array(st.per_case), data[tag + "/per_case"]), kind
        rates[kind] = st.rate
    assert rates["topk"] >= rates["retrieval"] > rates["streaming"]
    assert rates["retrieval"] - rates["streaming"] >= 0.3


def test_full_budget_self_draft_accepts_everything(P):
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=4, head_dim=8, d_ff=32, vocab_size=40, max_seq=128)
    w = P.generate_weights(cfg, 5)
    prefix = [1, 2, 3, 4, 5, 6, 7, 8]
    s = P.SingleLevelSession(w, P.FullCache.from_config(cfg), w, prefix, gamma=3, temperature=0.0)
    out, stats = s.generate(len(prefix) + 9, seed=0)
    assert stats.rate == 1.0
    assert out == P.autoregressive_generate(w, prefix, len(prefix) + 9, 0.0, 0)


def test_rerun_same_seed_same_stats(P, needle):
    target, draft, prompts = needle

    def run():
        cache = P.StreamingCache.from_config(draft.config, P.StreamingConfig(n_sink=2, budget=6))
        s = P.SingleLevelSession(draft, cache, target, prompts[9][:40], gamma=3, temperature=0.6)
        return s.generate(48, seed=3)

    (o1, s1), (o2, s2) = run(), run()
    assert o1 == o2 and (s1.proposed, s1.accepted, s1.rounds) == (s2.proposed, s2.accepted, s2.rounds)


def test_hierarchical_pairing_reports_both_levels(P, needle):
    target, draft, prompts = needle
    kw = dict(draft=draft, gamma=2, gamma2=3, gen_tokens=6, temperature=0.7, seed=2,
              streaming=P.StreamingConfig(n_sink=2, budget=10), retrieval=P.RetrievalConfig(chunk_size=4, budget=8))
    r1 = P.measure_acceptance("hierarchical", target, prompts[:2], **kw)
    r2 = P.measure_acceptance("hierarchical", target, prompts[:2], **kw)
    assert r1["inner"].rate == r2["inner"].rate and r1["outer"].rate == r2["outer"].rate
    assert r1["outer"].proposed > 0 and len(r1["inner"].per_case) == 2


def test_single_level_contract_errors(P, needle):
    target, draft, prompts = needle
    with pytest.raises(ValueError):
        P.SingleLevelSession(target, P.FullCache.from_config(target.config), target, prompts[0], 0, 0.0)
    with pytest.raises(P.ContractError):   # retrieval drafting needs the verify weights
        P.SingleLevelSession(draft, P.RetrievalCache.from_config(draft.config, P.RetrievalConfig(chunk_size=8,
                                                                                                budget=16)),
                             target, prompts[0], 2, 0.0)
    s = P.SingleLevelSession(target, P.FullCache.from_config(target.config), target, prompts[0][:10], 2, 0.0)
    with pytest.raises(ValueError):
        s.generate(10)


def test_attention_probe_matches_bruteforce(P):
    """ForwardRecorder(record_probs=True) / attention_probe (model.py:208-243,
    381-393) against an fp64 softmax recomputed from the recorded post-RoPE
    query and the cached bf16 keys; full and StreamingLLM caches."""
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=32, d_ff=96, vocab_size=64, max_seq=256)
    w = P.generate_weights(cfg, 17)
    prompt = np.random.default_rng(3).integers(1, 64, 90).tolist()
    for cache in (P.FullCache.from_config(cfg), P.StreamingCache.from_config(cfg, P.StreamingConfig(n_sink=4,
                                                                                                     budget=24))):
        rec = P.ForwardRecorder(record_probs=True)
        P.prefill(w, prompt, cache, rec)
        qs = rec.last_queries
        for li in range(cfg.n_layers):
            for h in range(cfg.n_heads):
                pr = P.attention_probe(rec, li, h)
                assert pr.query_position == len(prompt) - 1
                assert abs(float(pr.weights.sum()) - 1.0) < 1e-5
                kv = h // (cfg.n_heads // cfg.n_kv_heads)
                if cache.kind == 0:
                    slots = pr.positions
                else:
                    pos = cache.pos[li].cpu().numpy()
                    slots = np.array([int(np.nonzero(pos == p)[0][0]) for p in pr.positions])
                K = cache.k[li, kv, torch.as_tensor(slots, device="cuda")].float().cpu().numpy().astype(np.float64)
                s = K @ qs[li][h].astype(np.float64) / np.sqrt(cfg.head_dim)
                ref = np.exp(s - s.max())
                ref /= ref.sum()
                assert np.abs(pr.weights - ref).max() < 1e-6, (type(cache).__name__, li, h)
            if cache.kind == 1:   # StreamingLLM exposure: the 4 sinks + the last budget - sinks = 20 positions
                assert sorted(rec.positions[li].tolist()) == list(range(4)) + list(range(len(prompt) - 20,
                                                                                         len(prompt)))
    with pytest.raises(ValueError):
        P.attention_probe(P.ForwardRecorder(), 0, 0)


def test_recovery_analytics_match_reference(P, golden_single, needle):
    """sparsity_recovery / locality_recovery (analytics.py:36-106) on the
    planted-needle model against the reference's own values."""
    data, meta = golden_single
    target, _, prompts = needle
    m = meta["recovery"]
    sp = P.sparsity_recovery(target, prompts[m["sparsity_prompt"]], m["sparsity_budget"])
    assert np.allclose(sp, data["recovery/bf16/sparsity"], rtol=1e-4, atol=1e-5)
    lc = P.locality_recovery(target, prompts[m["locality_prompt"]], m["locality_budget"], horizon=m["horizon"])
    assert np.allclose(lc.frozen, data["recovery/bf16/frozen"], rtol=1e-4, atol=1e-5)
    assert np.allclose(lc.fresh, data["recovery/bf16/fresh"], rtol=1e-4, atol=1e-5)


def _h2o_row(qpos, positions):
    """deterministic unnormalised attention mass per exposed position (independent
    of which other entries are exposed), as in the reference's replay harness"""
    p = positions.astype(np.float64)
    return 1.0 / (1.0 + np.abs(qpos - p)) + 0.05 * ((positions * 40503) % 89) / 89.0


@pytest.mark.parametrize("policy", ["h2o", "topk"])
def test_rollback_replay_h2o_topk(P, policy):
    """Rollback soundness (tests/test_caches.py:416-435, acceptance criterion
    C6) for the two analytics policies: a cache driven through random
    speculate / commit / rollback rounds exposes exactly what a fresh cache fed
    only the committed history (same commit batching) exposes."""
    L, KVH, DH = 2, 2, 8

    def make():
        if policy == "h2o":
            return P.H2OCache(L, KVH, DH, P.H2OConfig(budget=9, recent_window=3), 512)
        return P.TopKCache(L, KVH, DH, 512, budget=7)

    def append_one(c, pos):
        for layer in range(L):
            base = np.arange(KVH * DH, dtype=np.float32).reshape(KVH, DH)
            k = (np.float32(0.001) * base + np.float32(pos + 0.01 * layer))[None]
            c.append(layer, k, -k)
            if c.wants_attention:
                pe = c.exposed_positions(layer)
                c.observe_attention(layer, _h2o_row(pos, pe).reshape(1, 1, 1, -1), np.array([pos]))

    def state(c):
        out = []
        for layer in range(L):
            K, V, pos, _ = c.expose(layer)
            out.append((K, V, pos))
        return out

    for trial in range(25):
        rng = np.random.default_rng(1000 + trial)
        live, oracle = make(), make()
        for c in (live, oracle):
            for p_ in range(12):
                append_one(c, p_)
            c.commit(12)
        committed, marks = 12, []
        for _ in range(8):
            n_spec = int(rng.integers(1, 5))
            for i in range(n_spec):
                append_one(live, committed + i)
            keep = int(rng.integers(0, n_spec + 1))
            live.rollback_to(committed + keep)
            live.commit(committed + keep)
            committed += keep
            marks.append(committed)
        pos = 12
        for mark in marks:
            while pos < mark:
                append_one(oracle, pos)
                pos += 1
            oracle.commit(mark)
        for (K1, V1, p1), (K2, V2, p2) in zip(state(live), state(oracle)):
            assert np.array_equal(p1, p2) and np.array_equal(K1, K2) and np.array_equal(V1, V2), (policy, trial)
        if policy == "h2o":
            for layer in range(L):
                assert len(live.exposed_positions(layer)) <= 9


def test_needle_criterion_with_own_fixtures(P):
    """Acceptance criterion 3 end to end with this package's own fixtures
    (host_analysis.needle_corpus / planted_attention_weights) instead of the
    reference-generated ones: top-k >= retrieval > streaming, gap >= 0.3."""
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=8, d_ff=32, vocab_size=260, max_seq=512,
                        rope_theta=1e8)
    corpus = P.needle_corpus(96, 30, seed=11)
    w = P.planted_attention_weights(cfg, 96, len(corpus[0].needle_positions), strength=0.8, answer_token=ord("A"),
                                    seed=11)
    prompts = [c.tokens for c in corpus]
    kw = dict(gamma=3, temperature=0.0, gen_tokens=8, seed=3, streaming=P.StreamingConfig(n_sink=4, budget=32),
              retrieval=P.RetrievalConfig(chunk_size=16, budget=32), topk_budget=32)
    rate = {k: P.measure_acceptance("self:" + k, w, prompts, **kw)["self"].rate
            for k in ("topk", "retrieval", "streaming")}
    assert rate["topk"] >= rate["retrieval"] > rate["streaming"], rate
    assert rate["retrieval"] - rate["streaming"] >= 0.3, rate


def test_self_speculation_head_dim_128(P):
    """StreamingLLM and H2O self-speculation on a head_dim-128 model: the
    streaming / H2O views run on the tensor-core attention (128-key splits),
    the streaming draft's captured one-token step with run-time positions
    (HsStep.dyn) included.  Checks: StreamingCache decode logits vs the CPU
    oracle's StreamingCache; greedy sessions == autoregressive (lossless);
    graph replay bit-identical to direct forwards."""
    from oracle import hs_oracle as O
    from paper_2404_11912_b200 import speculation as S
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=128, d_ff=344, vocab_size=512, max_seq=1024)
    w = P.plant_successor(P.generate_weights(cfg, 21, tied_head=False), 4, 0.8)
    prompt = np.random.default_rng(5).integers(1, 512, 300).tolist()
    # decode over a sink + window view vs the oracle (bf16 storage model)
    om = O.OModel(O.OConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__}),
                  O.round_weights_bf16(w.tensors), False)
    sc = P.StreamingCache.from_config(cfg, P.StreamingConfig(n_sink=4, budget=64))
    oc = O.OStreamingCache(2, 2, 128, 4, 64, kv_bf16=True)
    P.prefill(w, prompt[:200], sc)
    O.prefill(om, prompt[:200], oc)
    for tk in prompt[200:206]:
        got = P.decode_step(w, tk, sc)
        ref = O.decode_step(om, tk, oc)
        assert np.allclose(got, ref, rtol=1e-4, atol=1e-4 * np.abs(ref).max())
    ar = P.autoregressive_generate(w, prompt, 360, 0.0, 0)
    res = {}
    for kind in ("streaming", "h2o"):
        for graphs in ((False, True) if kind == "streaming" else (True,)):
            S.USE_GRAPHS = graphs
            try:
                cache = (P.StreamingCache.from_config(cfg, P.StreamingConfig(n_sink=4, budget=64)) if kind == "streaming"
                         else P.H2OCache.from_config(cfg, P.H2OConfig(budget=64, recent_window=16)))
                s = P.SingleLevelSession(w, cache, w, prompt, gamma=3, temperature=0.0)
                out, st = s.generate(360, seed=0)
            finally:
                S.USE_GRAPHS = True
            assert out == ar, (kind, graphs)
            assert st.accepted > 0
            res[(kind, graphs)] = (out, st.proposed, st.accepted, st.rounds)
    assert res[("streaming", False)] == res[("streaming", True)]
