"""End-to-end parity on the B200 (`-m gpu`): forwards, caches and the
hierarchical loop against the reference's golden fixtures (bf16 storage
model) and the CPU oracle."""

from __future__ import annotations

import io
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2404_11912_b200 as pkg
    return pkg


def small_config(P, **kw):
    base = dict(n_layers=2, n_heads=4, n_kv_heads=4, head_dim=8, d_ff=32, vocab_size=40, max_seq=128)
    base.update(kw)
    return P.ModelConfig(**base)


def bf16_weights(P, w):
    from oracle.hs_oracle import bf16_round
    t = {n: (x.copy() if "norm" in n else bf16_round(x)) for n, x in w.tensors.items()}
    return P.ModelWeights(w.config, t, w.tied_head).validate()


# ---------------------------------------------------------------------------
# forward

def test_forward_matches_reference_bf16(P, golden):
    data, meta = golden
    for c in meta["forward_cases"]:
        cfg = P.ModelConfig(**c["cfg"])
        w = bf16_weights(P, P.generate_weights(cfg, c["seed"], c["tied"]))
        cache = P.FullCache.from_config(cfg)
        rec = P.ForwardRecorder()
        lg = P.prefill(w, c["prefill"], cache, rec)
        ref = data[f"fwd/{c['name']}/bf16/prefill"]
        assert np.allclose(lg, ref, rtol=1e-4, atol=1e-5), c["name"]
        assert np.allclose(np.stack(rec.last_queries), data[f"fwd/{c['name']}/bf16/q_last"], rtol=1e-4, atol=1e-5)
        rows = np.stack([P.decode_step(w, tk, cache) for tk in c["decode"]])
        assert np.allclose(rows, data[f"fwd/{c['name']}/bf16/decode"], rtol=1e-4, atol=1e-5)
        assert (np.argmax(rows, -1) == np.argmax(data[f"fwd/{c['name']}/bf16/decode"], -1)).all()


def test_chunk_equals_step_sequence_bitwise(P):
    cfg = small_config(P)
    w = P.generate_weights(cfg, 11)
    c1 = P.FullCache.from_config(cfg)
    P.prefill(w, [1, 2, 3, 4, 5, 6, 7, 8], c1)
    c2 = c1.clone()
    chunk = P.decode_chunk(w, [9, 10, 11], c1)
    steps = np.stack([P.decode_step(w, tk, c2) for tk in (9, 10, 11)])
    assert np.array_equal(chunk, steps)
    # across the 8-row block boundary (multi-block path vs single-row steps)
    toks = list(range(12, 32))
    chunk = P.decode_chunk(w, toks, c1)
    steps = np.stack([P.decode_step(w, tk, c2) for tk in toks])
    assert np.array_equal(chunk, steps)
    assert torch.equal(c1.k, c2.k) and torch.equal(c1.v, c2.v)


def test_cfg1_prefill_and_queries(P, golden):
    """Config 1 (4K context, untied): last prefill row and the builder's
    queries match the reference within fp32-level tolerance."""
    data, meta = golden
    c = meta["cfg1"]
    cfg = P.ModelConfig(**c["target"])
    w = bf16_weights(P, P.generate_weights(cfg, 1, tied_head=False))
    prompt = np.random.default_rng(0).integers(1, 256, 4096).tolist()
    cache = P.FullCache.from_config(cfg)
    rec = P.ForwardRecorder()
    lg = P.prefill(w, prompt, cache, rec)
    ref_lg, ref_q = data["cfg1/bf16/prefill_last"], data["cfg1/bf16/q_last"]
    e_lg = np.abs(lg[-1] - ref_lg).max() / np.abs(ref_lg).max()
    e_q = np.abs(np.stack(rec.last_queries) - ref_q).max() / np.abs(ref_q).max()
    print(f"cfg1 prefill: logits max err / max |logit| = {e_lg:.3g}, queries {e_q:.3g}")
    # fp32 accumulation (GPU) vs fp64 accumulation rounded to fp32 (reference)
    # over 4,096 positions, 2 layers: a few 1e-7 of the largest value
    # (observed 3.6e-5 / 1.7e-5: beyond fp32 accumulation noise because a
    # last-bit difference in a K/V projection occasionally flips its bf16
    # rounding in the cache -- a 2^-8 relative step -- which the reference's
    # bf16-rounding cache then does not share; the north star's bar for
    # attention outputs is 2e-2)
    assert e_lg < 1e-4 and e_q < 1e-4, (e_lg, e_q)
    assert lg[-1].argmax() == ref_lg.argmax()


def test_errors(P):
    cfg = small_config(P)
    w = P.generate_weights(cfg, 11)
    cache = P.FullCache.from_config(cfg)
    with pytest.raises(ValueError):
        P.prefill(w, [], cache)
    with pytest.raises(P.CapacityError):
        P.prefill(w, [1] * (cfg.max_seq + 1), cache)
    with pytest.raises(ValueError):
        P.decode_step(w, 1, P.FullCache.from_config(cfg))


# ---------------------------------------------------------------------------
# caches (reference tests/test_caches.py semantics on the device caches)

def _kv_for(pos, layer, kvh, dh):
    base = np.arange(kvh * dh, dtype=np.float32).reshape(kvh, dh)
    k = np.float32(0.001) * base + np.float32(pos + 0.01 * layer)
    return k[None], -k[None]


def _fill(cache, n, commit=True):
    for pos in range(cache.frontier, cache.frontier + n):
        for layer in range(cache.n_layers):
            k, v = _kv_for(pos, layer, cache.n_kv_heads, cache.head_dim)
            cache.append(layer, k, v)
    if commit:
        cache.commit(cache.frontier)


def test_streaming_exposure_examples(P):
    s = P.StreamingCache(2, 2, 8, P.StreamingConfig(n_sink=4, budget=10))
    _fill(s, 100)
    assert s.exposed_positions(0).tolist() == list(range(4)) + list(range(94, 100))
    s = P.StreamingCache(2, 2, 8, P.StreamingConfig(n_sink=2, budget=6))
    _fill(s, 10)
    assert s.to_json()["layers"][0]["exposed_positions"] == [0, 1, 6, 7, 8, 9]
    _fill(s, 3, commit=False)
    assert len(s.exposed_positions(0)) <= 6
    with pytest.raises(P.ContractError):
        s.rollback_to(5)


def _replay(P, O, make_pair, setup_pair, trials, seed0):
    """Random speculate/commit/rollback schedules (tests/cache_replay.py)
    applied to the device cache and the oracle cache in lockstep."""
    for trial in range(trials):
        rng = np.random.default_rng(seed0 + trial)
        dev, orc = make_pair()
        setup_pair(dev, orc)
        committed = dev.frontier
        for _ in range(8):
            n_spec = int(rng.integers(1, 5))
            for i in range(n_spec):
                for layer in range(dev.n_layers):
                    k, v = _kv_for(committed + i, layer, dev.n_kv_heads, dev.head_dim)
                    dev.append(layer, k, v)
                    orc.append(layer, k, v)
            keep = int(rng.integers(0, n_spec + 1))
            for c in (dev, orc):
                c.rollback_to(committed + keep)
                c.commit(committed + keep)
            committed += keep
            for layer in range(dev.n_layers):
                K, V, pos, _ = dev.expose(layer)
                oK, oV, opos = orc.view(layer)
                assert np.array_equal(pos, opos), trial
                assert np.array_equal(K, oK) and np.array_equal(V, oV), trial


def test_rollback_replay_full_streaming_retrieval(P):
    from oracle import hs_oracle as O

    def fill_both(d, o):
        for pos in range(12):
            for layer in range(d.n_layers):
                k, v = _kv_for(pos, layer, d.n_kv_heads, d.head_dim)
                d.append(layer, k, v)
                o.append(layer, k, v)
        d.commit(12)
        o.commit(12)

    _replay(P, O, lambda: (P.FullCache(2, 2, 4 * 2, 512), O.OFullCache(2, 2, 8, 512, kv_bf16=True)),
            fill_both, 20, 1000)
    _replay(P, O, lambda: (P.StreamingCache(2, 2, 8, P.StreamingConfig(n_sink=2, budget=9)),
                           O.OStreamingCache(2, 2, 8, 2, 9, kv_bf16=True)), fill_both, 20, 1000)

    src_d = P.FullCache(2, 2, 8, 512)
    src_o = O.OFullCache(2, 2, 8, 512, kv_bf16=True)
    fill_both(src_d, src_o)
    for pos in range(12, 16):
        for layer in range(2):
            k, v = _kv_for(pos, layer, 2, 8)
            src_d.append(layer, k, v)
            src_o.append(layer, k, v)
    src_d.commit(16)
    src_o.commit(16)
    qs = [np.random.default_rng(7).normal(0, 1, (2, 8)).astype(np.float32) for _ in range(2)]

    def build_both(d, o):
        d.build(src_d, qs, 16)
        o.build(src_o, qs, 16)

    _replay(P, O, lambda: (P.RetrievalCache(2, 2, 8, P.RetrievalConfig(chunk_size=4, budget=8)),
                           O.ORetrievalCache(2, 2, 8, 4, 8, kv_bf16=True)), build_both, 40, 2000)


def test_should_rebuild_truth_table(P):
    cfg = P.RetrievalConfig(rebuild_stride=128, rebuild_accept_threshold=0.8, rolling_window=4)
    r = P.RollingAcceptance(4)
    assert P.should_rebuild(cfg, 128, r)
    r.push(1.0)
    assert not P.should_rebuild(cfg, 0, r)
    for _ in range(4):
        r.push(0.5)
    assert P.should_rebuild(cfg, 0, r)


# ---------------------------------------------------------------------------
# the hierarchical loop

def _small_session(P, kw, mode="bf16"):
    kw = dict(kw)
    cfg = small_config(P)
    target = P.generate_weights(cfg, 11)
    draft = P.generate_weights(small_config(P, n_layers=1), 12)
    if mode == "bf16":
        target, draft = bf16_weights(P, target), bf16_weights(P, draft)
    prefix_len = kw.pop("prefix_len", 24)
    prefix = np.random.default_rng(99).integers(1, cfg.vocab_size, prefix_len).tolist()
    spec = P.SpecConfig(target_len=kw.pop("target_len", prefix_len + 12), gamma1=kw.pop("gamma1", 2),
                        gamma2=kw.pop("gamma2", 4), temperature=kw.pop("temperature", 0.0), seed=5,
                        streaming=P.StreamingConfig(n_sink=2, budget=12),
                        retrieval=P.RetrievalConfig(chunk_size=kw.pop("chunk", 4), budget=kw.pop("budget", 16),
                                                    **kw))
    return target, draft, prefix, spec


def test_small_sessions_match_reference(P, golden):
    """Token streams, level labels and acceptance counters equal the
    reference run (bf16 storage model) -- greedy and sampled."""
    data, meta = golden
    levels = ["draft", "retrieval", "corrected", "bonus"]
    for i, kw in enumerate(meta["small_sessions"]):
        target, draft, prefix, spec = _small_session(P, kw)
        out, tr = P.HierarchicalSession(target, draft, prefix, spec).generate()
        tag = f"sess/{i}/bf16"
        assert out == data[tag + "/tokens"].tolist(), (i, kw)
        s = tr.summary()
        assert [s["inner"]["proposed"], s["inner"]["accepted"], s["inner"]["rounds"], s["outer"]["proposed"],
                s["outer"]["accepted"], s["outer"]["rounds"]] == data[tag + "/stats"].tolist(), (i, kw)
        assert [levels.index(r["level"]) for r in tr.records] == data[tag + "/rec_level"].tolist()


@pytest.mark.parametrize("budget,chunk", [(8, 4), (16, 4), (32, 4)])
def test_greedy_losslessness_across_budgets(P, budget, chunk):
    target, draft, prefix, spec = _small_session(P, dict(budget=budget, chunk=chunk, prefix_len=20, target_len=36),
                                                 mode="plain")
    out, _ = P.hierarchical_generate(target, draft, prefix, spec)
    assert out == P.autoregressive_generate(target, prefix, spec.target_len, 0.0, 0)


def test_rebuild_fires_and_stays_lossless(P):
    target, draft, prefix, spec = _small_session(
        P, dict(budget=8, chunk=4, prefix_len=20, target_len=44, rebuild_stride=6, rolling_window=4), mode="plain")
    session = P.HierarchicalSession(target, draft, prefix, spec)
    out, _ = session.generate()
    assert session.rebuilds >= 1
    assert out == P.autoregressive_generate(target, prefix, spec.target_len, 0.0, 0)


def test_autoregressive_matches_reference(P, golden):
    data, meta = golden
    from oracle import hs_oracle as O
    for i, c in enumerate(meta["ar_cases"]):
        w = P.generate_weights(small_config(P), c["seed"])
        out = P.autoregressive_generate(w, [1, 2, 3], 14, c["temperature"], seed=c["rng_seed"])
        # plain-weights golden; bf16 weights may flip near-ties, so compare to the bf16 oracle
        ow = O.OModel(O.OConfig(**{k: getattr(w.config, k) for k in w.config.__dataclass_fields__}),
                      O.round_weights_bf16(w.tensors), True)
        assert out == O.ar_generate(ow, [1, 2, 3], 14, c["temperature"], seed=c["rng_seed"], kv_bf16=True)


def test_adversarial_draft_progress(P):
    target, draft, prefix, spec = _small_session(P, dict(temperature=0.5, target_len=40), mode="plain")
    draft.tensors["embedding"][:] = 0.0
    draft._runtime = None
    out, trace = P.hierarchical_generate(target, draft, prefix, spec)
    assert len(out) == spec.target_len
    assert trace.outer.rounds <= spec.target_len - len(prefix)
    assert len(trace.records) == spec.target_len - len(prefix)


def test_trace_jsonl_and_accounting(P):
    target, draft, prefix, spec = _small_session(P, dict(temperature=0.7, target_len=44), mode="plain")
    _, trace = P.hierarchical_generate(target, draft, prefix, spec)
    assert trace.inner.accepted + trace.inner.rejected == trace.inner.proposed
    buf = io.StringIO()
    trace.to_jsonl(buf)
    lines = [json.loads(x) for x in buf.getvalue().splitlines()]
    assert len(lines) == len(trace.records)
    assert {r["level"] for r in lines} <= {"draft", "retrieval", "corrected", "bonus"}


def test_cache_coherence_after_generation(P):
    target, draft, prefix, spec = _small_session(P, dict(target_len=34), mode="plain")
    session = P.HierarchicalSession(target, draft, prefix, spec)
    out, _ = session.generate()
    pos = session.full_lane.cache.exposed_positions(0)
    assert np.array_equal(pos, np.arange(len(pos)))
    assert session.full_lane.cache.committed == len(pos) <= len(out)


def test_single_round_api_matches_oracle(P):
    """draft_round / inner_speculate / outer_verify with an external rng keep
    the caller's Generator at the reference's stream position."""
    target, draft, prefix, spec = _small_session(P, dict(temperature=0.9), mode="plain")
    s = P.HierarchicalSession(target, draft, prefix, spec)
    rng = np.random.default_rng(11)
    x_hat, p_hats, _ = P.inner_speculate(s.retr_lane, s.draft_lane, s.committed, spec, rng)
    emitted, labels, accepted, _ = P.outer_verify(s.full_lane, s.committed, x_hat, p_hats, 0.9, rng)
    assert emitted[:accepted] == x_hat[:accepted]
    assert len(emitted) == accepted + 1 <= len(x_hat) + 1
    # same calls through the oracle consume the same number of uniforms
    from oracle import hs_oracle as O
    mk = lambda w: O.OModel(O.OConfig(**{k: getattr(w.config, k) for k in w.config.__dataclass_fields__}),
                            O.round_weights_bf16(w.tensors), w.tied_head)
    os_ = O.OSession(mk(target), mk(draft), prefix, O.OSpec(target_len=spec.target_len, gamma1=2, gamma2=4,
                     temperature=0.9, n_sink=2, stream_budget=12, chunk=4, retr_budget=16), kv_bf16=True)
    r2 = np.random.default_rng(11)
    tr = O.OTrace()
    ox, oph, _ = os_._inner(r2, tr)
    assert ox == x_hat


def _delta_consistent(gpu_imp, ref_imp, ref_scores, delta):
    """True iff the GPU's importance list can be the reference's selection
    under score perturbations of at most `delta` per chunk: every chunk only
    one side chose sits within 2*delta of the reference's selection threshold,
    and the GPU's order never ranks a chunk above one whose reference score
    is higher by more than 2*delta (caches.py:474-486, ties to the lower id)."""
    tol = 2.0 * delta
    thr = min(ref_scores[c] for c in ref_imp[1:])
    for c in set(gpu_imp) ^ set(ref_imp):
        if abs(ref_scores[c] - thr) > tol:
            return False
    rest = [ref_scores[c] for c in gpu_imp[1:]]
    suffix = -np.inf
    for v in reversed(rest):
        if v < suffix - tol:
            return False
        suffix = max(suffix, v)
    return gpu_imp[0] == ref_imp[0]   # the pinned last chunk


@pytest.mark.slow
def test_cfg1_greedy_and_sampled(P, golden):
    """BASELINE config 1 (the reference's own CPU-runnable configuration).

    Against the reference's goldens:
    * initial build: the GPU's top-k ids, importance order and victim FIFO
      are bit-exact against the oracle's selection on the GPU's own keys and
      query; against the reference's ids (whose cached keys differ from the
      GPU's by fp32 accumulation and the occasional bf16 rounding flip) they
      are identical, or every difference is a near-tie within twice the
      measured score perturbation (reference scores from make_golden.py);
    * T = 0: the 64-token stream and per-level counts equal the reference's.
    On identical inputs (the CPU oracle twin of the GPU session's state
    after prefill and build, tests/_twin.py):
    * T = 0.6 at the fixed seed: inner and outer acceptance within +-1%
      (and the 64-token streams, labels and counts identical)."""
    from oracle import hs_oracle as O
    from tests._twin import oracle_twin
    data, meta = golden
    c = meta["cfg1"]
    tw = bf16_weights(P, P.generate_weights(P.ModelConfig(**c["target"]), 1, tied_head=False))
    dw = bf16_weights(P, P.generate_weights(P.ModelConfig(**c["draft"]), 2, tied_head=False))
    prompt = np.random.default_rng(0).integers(1, 256, 4096).tolist()
    for temp in (0.0, 0.6):
        spec = P.SpecConfig(target_len=4096 + 64, gamma1=2, gamma2=4, temperature=temp, seed=0,
                            streaming=P.StreamingConfig(n_sink=4, budget=256),
                            retrieval=P.RetrievalConfig(chunk_size=8, budget=256))
        sess = P.HierarchicalSession(tw, dw, prompt, spec)
        tag = f"cfg1/bf16/T{temp}"
        tab = sess.retr_lane.cache.table
        imp0 = tab.selected
        rc = sess.retr_lane.cache
        q = sess.full_lane.recorder.stash.cpu().numpy()
        ref_imp = data[tag + "/importance0"].tolist()
        ref_sc = data[tag + "/scores0"]
        for li in range(2):
            # exact: the oracle's selection on the GPU's inputs
            K = sess.full_lane.cache.k[li, :, :4095].permute(1, 0, 2).float().cpu().numpy()
            bounds, osc = O.chunk_scores(K, q[li], 8, 4)
            _, oimp = O.select_chunks(osc, 32, False)
            assert imp0[li] == oimp, li
            # same fp64 arithmetic up to the order of the 8-key chunk sums
            assert np.allclose(tab.scores[li], osc, rtol=1e-12, atol=1e-15 * np.abs(osc).max()), li
            pos = rc.pos[li, :rc.n_sel].cpu().numpy()
            vict = [p for ci in reversed(oimp) for p in range(int(bounds[ci]), int(bounds[ci + 1]))]
            assert pos[rc.ring[li, :rc.n_sel].cpu().numpy()].tolist() == vict, li
            # vs the reference's own build
            delta = float(np.abs(tab.scores[li] - ref_sc[li]).max())
            same = imp0[li] == ref_imp[li]
            print(f"cfg1 T={temp} layer {li}: ids {'identical' if same else 'differ'} to the reference; "
                  f"max |score - ref score| = {delta:.3g}")
            assert same or _delta_consistent(imp0[li], ref_imp[li], ref_sc[li], delta), li
        twin = None
        if temp > 0:
            mk = lambda w: O.OModel(O.OConfig(**{k: getattr(w.config, k) for k in w.config.__dataclass_fields__}),
                                    O.round_weights_bf16(w.tensors), w.tied_head)
            twin = oracle_twin(O, sess, mk(tw), mk(dw),
                               O.OSpec(target_len=4096 + 64, gamma1=2, gamma2=4, temperature=temp, seed=0,
                                       n_sink=4, stream_budget=256, chunk=8, retr_budget=256))
        out, tr = sess.generate()
        st = data[tag + "/stats"].tolist()
        s = tr.summary()
        agree = next((i for i, (a, b) in enumerate(zip(out[4096:], data[tag + "/tokens"].tolist())) if a != b), 64)
        print(f"cfg1 T={temp}: GPU {s}; reference stats {st}; streams agree with the reference on {agree}/64")
        if temp == 0.0:
            assert out[4096:] == data[tag + "/tokens"].tolist()
            assert [s["inner"]["proposed"], s["inner"]["accepted"], s["inner"]["rounds"],
                    s["outer"]["proposed"], s["outer"]["accepted"], s["outer"]["rounds"]] == st[:6]
        else:
            oout, otr = twin.generate(seed=0)
            os_ = otr.summary()
            print(f"cfg1 T={temp}: oracle twin {os_}")
            assert abs(s["inner"]["rate"] - os_["inner"]["rate"]) <= 0.01, (s, os_)
            assert abs(s["outer"]["rate"] - os_["outer"]["rate"]) <= 0.01, (s, os_)
            assert out == oout and s == os_
            assert [r["level"] for r in tr.records] == [r["level"] for r in otr.records]


def _desk(P, seed):
    t = P.generate_weights(P.ModelConfig(n_layers=4, n_heads=8, n_kv_heads=4, head_dim=16, d_ff=256, vocab_size=260,
                                         max_seq=1024), seed=seed, tied_head=False)
    d = P.generate_weights(P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=4, head_dim=16, d_ff=128, vocab_size=260,
                                         max_seq=1024), seed=1000 + seed, tied_head=False)
    return t, d


def test_sampled_acceptance_rates(P):
    """North-star criterion: at T=0.6 with fixed seeds the GPU loop's inner
    and outer acceptance rates agree with the CPU oracle within +-1%
    (aggregated over 24 (seed, prompt) runs of 48 tokens, desk-scale models
    of the reference's conftest with untied heads)."""
    from oracle import hs_oracle as O
    mk = lambda w: O.OModel(O.OConfig(**{k: getattr(w.config, k) for k in w.config.__dataclass_fields__}),
                            O.round_weights_bf16(w.tensors), w.tied_head)
    g = np.zeros(4)
    o = np.zeros(4)
    for i in range(24):
        tw, dw = _desk(P, i)
        prompt = np.random.default_rng(i).integers(1, 260, 192).tolist()
        spec = P.SpecConfig(target_len=240, gamma1=2, gamma2=4, temperature=0.6, seed=i,
                            streaming=P.StreamingConfig(n_sink=4, budget=64),
                            retrieval=P.RetrievalConfig(chunk_size=8, budget=64))
        _, tr = P.HierarchicalSession(tw, dw, prompt, spec).generate()
        g += [tr.inner.accepted, tr.inner.proposed, tr.outer.accepted, tr.outer.proposed]
        os_ = O.OSession(mk(tw), mk(dw), prompt, O.OSpec(target_len=240, gamma1=2, gamma2=4, temperature=0.6, seed=i,
                         n_sink=4, stream_budget=64, chunk=8, retr_budget=64), kv_bf16=True)
        _, otr = os_.generate()
        o += [otr.inner[1], otr.inner[0], otr.outer[1], otr.outer[0]]
    assert abs(g[0] / g[1] - o[0] / o[1]) <= 0.01, (g, o)
    assert abs(g[2] / g[3] - o[2] / o[3]) <= 0.01, (g, o)


@pytest.mark.parametrize("head_dim", [64, 128])
def test_planted_greedy_stream_and_acceptance_match_oracle(P, head_dim):
    """Non-degenerate acceptance (random-init greedy is vacuous):
    models with a planted successor channel accept most speculations, and the
    GPU loop's greedy stream and per-level accept counts equal the oracle's
    exactly, rebuilds included.  head_dim 128 runs the target on the
    tensor-core attention with RoPE + append fused into it."""
    from oracle import hs_oracle as O
    mk = lambda w: O.OModel(O.OConfig(**{k: getattr(w.config, k) for k in w.config.__dataclass_fields__}),
                            O.round_weights_bf16(w.tensors), w.tied_head)
    tc = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=head_dim, d_ff=344, vocab_size=512,
                       max_seq=2048)
    dc = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=64, d_ff=172, vocab_size=512, max_seq=2048)
    tw = bf16_weights(P, P.plant_successor(P.generate_weights(tc, 5, tied_head=False), 9, 0.9))
    dw = bf16_weights(P, P.plant_successor(P.generate_weights(dc, 6, tied_head=False), 9, 0.9))
    prompt = np.random.default_rng(3).integers(1, 512, 1200).tolist()
    spec = P.SpecConfig(target_len=1200 + 96, gamma1=2, gamma2=4, temperature=0.0, seed=0,
                        streaming=P.StreamingConfig(n_sink=4, budget=128),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=128, rebuild_stride=32))
    out, tr = P.HierarchicalSession(tw, dw, prompt, spec).generate()
    os_ = O.OSession(mk(tw), mk(dw), prompt, O.OSpec(target_len=1200 + 96, gamma1=2, gamma2=4, temperature=0.0,
                     seed=0, n_sink=4, stream_budget=128, chunk=8, retr_budget=128, rebuild_stride=32),
                     kv_bf16=True)
    oout, otr = os_.generate()
    assert out == oout
    assert [tr.inner.proposed, tr.inner.accepted] == otr.inner[:2]
    assert [tr.outer.proposed, tr.outer.accepted] == otr.outer[:2]
    assert tr.outer.rate > 0.6 and tr.inner.rate > 0.6, tr.summary()


def test_generate_continues_after_truncated_round(P):
    """bench.py extends target_len and calls generate() again; the lanes must
    stay resumable after a truncated final round and the greedy stream must
    still be the autoregressive one."""
    tc = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=64, d_ff=344, vocab_size=512, max_seq=1024)
    dc = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=64, d_ff=172, vocab_size=512, max_seq=1024)
    tw = P.plant_successor(P.generate_weights(tc, 5, tied_head=False), 9, 0.95)
    dw = P.plant_successor(P.generate_weights(dc, 6, tied_head=False), 9, 0.95)
    prompt = np.random.default_rng(4).integers(1, 512, 300).tolist()
    spec = P.SpecConfig(target_len=301, gamma1=2, gamma2=4, temperature=0.0, seed=0,
                        streaming=P.StreamingConfig(n_sink=4, budget=64),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=64, rebuild_stride=16))
    s = P.HierarchicalSession(tw, dw, prompt, spec)
    for n in (301, 303, 310, 311, 340):
        s.config.target_len = n
        out, _ = s.generate()
        assert len(out) == n
    assert out == P.autoregressive_generate(tw, prompt, 340, 0.0, 0)


def test_draft_step_graphs_match_direct_forwards(P):
    """The draft lane's captured one-token step (CUDA graph, run-time
    frontier via HsStep.dyn) gives the same session, bit for bit, as direct
    hs_forward calls."""
    from paper_2404_11912_b200 import speculation as S
    tc = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=64, d_ff=344, vocab_size=512, max_seq=2048)
    dc = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=4, head_dim=64, d_ff=172, vocab_size=512, max_seq=2048)
    tw = P.plant_successor(P.generate_weights(tc, 5, tied_head=False), 9, 0.8)
    dw = P.plant_successor(P.generate_weights(dc, 6, tied_head=False), 9, 0.8)
    prompt = np.random.default_rng(8).integers(1, 512, 700).tolist()
    res = []
    for graphs in (False, True):
        S.USE_GRAPHS = graphs
        try:
            spec = P.SpecConfig(target_len=700 + 90, gamma1=3, gamma2=5, temperature=0.7, seed=2,
                                streaming=P.StreamingConfig(n_sink=4, budget=96),
                                retrieval=P.RetrievalConfig(chunk_size=8, budget=128, rebuild_stride=40))
            s = P.HierarchicalSession(tw, dw, prompt, spec)
            out, tr = s.generate()
            res.append((out, tr.summary(), s.draft_lane.cache.k.clone(), s.draft_lane._front.clone()))
        finally:
            S.USE_GRAPHS = True
    assert res[0][0] == res[1][0] and res[0][1] == res[1][1]
    assert torch.equal(res[0][2], res[1][2]) and torch.equal(res[0][3], res[1][3])


@pytest.mark.parametrize("head_dim,split_at", [(64, 0), (128, 0), (128, 700)])
def test_gemm_prefill_matches_decode_path(P, head_dim, split_at):
    """Batched GEMM prefill (hs_prefill, >= 64 rows) against the row-exact
    decode path on the same prompt: logits within fp32 accumulation noise,
    same argmaxes, same cached K/V to bf16 rounding.  head_dim 128 runs the
    128-row tensor-core prefill attention (prefill_attn.cu), also as a second
    prefill appended to a non-empty cache (queries at positions >= 700)."""
    from paper_2404_11912_b200 import model as M
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=head_dim, d_ff=344, vocab_size=512,
                        max_seq=4096)
    w = P.generate_weights(cfg, 21, tied_head=False)
    prompt = np.random.default_rng(2).integers(1, 512, 1500).tolist()
    a, b = P.FullCache.from_config(cfg), P.FullCache.from_config(cfg)
    if split_at:
        la = np.concatenate([P.prefill(w, prompt[:split_at], a), P.prefill(w, prompt[split_at:], a)])
    else:
        la = P.prefill(w, prompt, a)                                          # GEMM prefill
    lb = M._host_rows(M.forward_device(w, prompt, b, None, prefill=False))    # decode-path rows
    # both paths are fp32-accurate, but K/V are stored in bf16: where the two
    # fp32 results straddle a rounding boundary the cached element differs by
    # one bf16 ulp (2^-8), which moves later logits by ~1e-4 relative
    assert np.allclose(la, lb, rtol=1e-4, atol=3e-4 * np.abs(lb).max())
    assert (np.argmax(la, -1) == np.argmax(lb, -1)).mean() > 0.999
    dk = (a.k[:, :, :1500].float() - b.k[:, :, :1500].float()).abs().max().item()
    assert dk <= 0.02 * b.k[:, :, :1500].float().abs().max().item()


@pytest.mark.parametrize("prompt_len,chunk,budget,stream,temp", [
    (1, 8, 64, 16, 0.0),        # one-token prompt: the build's n == 1 special case (speculation.py:305-308)
    (37, 16, 64, 32, 0.6),      # ragged last chunk, sampled
    (203, 8, 256, 64, 0.0),     # budget >= context: clamped build (all chunks)
    (1203, 16, 64, 48, 0.6),    # long, ragged, tiny budget, sampled
])
def test_edge_sessions_match_oracle(P, prompt_len, chunk, budget, stream, temp):
    """Edge geometries of the reference's build/stream rules, with
    non-degenerate acceptance: token stream, per-level accept counts and the
    initial build's chunk selection equal the oracle's."""
    from oracle import hs_oracle as O
    mk = lambda w: O.OModel(O.OConfig(**{k: getattr(w.config, k) for k in w.config.__dataclass_fields__}),
                            O.round_weights_bf16(w.tensors), w.tied_head)
    tc = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=32, d_ff=96, vocab_size=300, max_seq=2048)
    dc = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=32, d_ff=64, vocab_size=300, max_seq=2048)
    tw = bf16_weights(P, P.plant_successor(P.generate_weights(tc, 31, tied_head=False), 4, 0.85))
    dw = bf16_weights(P, P.plant_successor(P.generate_weights(dc, 32, tied_head=False), 4, 0.85))
    prompt = np.random.default_rng(prompt_len).integers(1, 300, prompt_len).tolist()
    n_gen = 48
    spec = P.SpecConfig(target_len=prompt_len + n_gen, gamma1=2, gamma2=4, temperature=temp, seed=7,
                        streaming=P.StreamingConfig(n_sink=4, budget=stream),
                        retrieval=P.RetrievalConfig(chunk_size=chunk, budget=budget, rebuild_stride=24))
    s = P.HierarchicalSession(tw, dw, prompt, spec)
    imp0 = s.retr_lane.cache.table.selected
    out, tr = s.generate()
    os_ = O.OSession(mk(tw), mk(dw), prompt, O.OSpec(target_len=prompt_len + n_gen, gamma1=2, gamma2=4,
                                                    temperature=temp, seed=7, n_sink=4, stream_budget=stream,
                                                    chunk=chunk, retr_budget=budget, rebuild_stride=24),
                     kv_bf16=True)
    oimp0 = [list(map(int, layer[2])) for layer in os_.builds[0][0]]   # (bounds, scores, importance) per layer
    oout, otr = os_.generate()
    assert out == oout
    assert [tr.inner.proposed, tr.inner.accepted, tr.outer.proposed, tr.outer.accepted] == \
        [otr.inner[0], otr.inner[1], otr.outer[0], otr.outer[1]]
    assert imp0 == oimp0


@pytest.mark.parametrize("temp", [0.6, 1.0])
def test_first_token_distribution_is_lossless(P, temp):
    """Acceptance criterion 2 on the device (tests/test_acceptance.py:67-138):
    the first token emitted by the two-level loop is distributed as the
    target model's own next-token distribution -- whatever the draft and the
    retrieval lane proposed.  3,000 sampled sessions cloned from one prefill,
    chi-square against p = softmax(full-lane logits / T) (bins with expected
    count < 5 pooled)."""
    from scipy.stats import chi2
    cfg_t = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=32, d_ff=96, vocab_size=24, max_seq=256)
    cfg_d = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=32, d_ff=64, vocab_size=24, max_seq=256)
    tw = P.plant_successor(P.generate_weights(cfg_t, 41, tied_head=False), 6, 0.6)
    dw = P.generate_weights(cfg_d, 42, tied_head=False)       # an unrelated draft: many rejections
    prompt = np.random.default_rng(5).integers(1, 24, 80).tolist()
    spec = P.SpecConfig(target_len=81, gamma1=2, gamma2=4, temperature=temp, seed=0,
                        streaming=P.StreamingConfig(n_sink=2, budget=16),
                        retrieval=P.RetrievalConfig(chunk_size=4, budget=16))
    base = P.HierarchicalSession(tw, dw, prompt, spec)
    logits = base.full_lane.frontier_logits.double().cpu().numpy()
    z = logits / temp
    p = np.exp(z - z.max())
    p /= p.sum()
    n = 3000
    counts = np.zeros(len(p))
    for i in range(n):
        s = base.clone()
        out, _ = s.generate(seed=1000 + i)
        counts[out[len(prompt)]] += 1
    exp_ = n * p
    big = exp_ >= 5
    obs = np.append(counts[big], counts[~big].sum())
    ex = np.append(exp_[big], exp_[~big].sum())
    keep = ex > 0
    stat = (((obs - ex) ** 2)[keep] / ex[keep]).sum()
    dof = int(keep.sum()) - 1
    assert chi2.sf(stat, dof) > 1e-4, (stat, dof, counts, exp_)


def test_greedy_equals_autoregressive_many_pairs(P):
    """Acceptance criterion 1 (tests/test_acceptance.py:36-58) at desk scale:
    greedy two-level decoding emits exactly the autoregressive tokens for 30
    (seed, prompt) pairs x retrieval budgets of 25 / 50 / 100 % of the
    context, with a planted target so the draft is right often but not
    always."""
    cfg_t = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=32, d_ff=96, vocab_size=64, max_seq=256)
    cfg_d = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=32, d_ff=64, vocab_size=64, max_seq=256)
    mismatches = []
    for i in range(30):
        tw = P.plant_successor(P.generate_weights(cfg_t, 100 + i, tied_head=False), 3 + i, 0.8)
        dw = P.plant_successor(P.generate_weights(cfg_d, 200 + i, tied_head=False), 3 + i, 0.8)
        plen = 48 + 4 * i
        prompt = np.random.default_rng(i).integers(1, 64, plen).tolist()
        ar = P.autoregressive_generate(tw, prompt, plen + 24, 0.0, 0)
        for frac in (0.25, 0.5, 1.0):
            budget = max(8, int(frac * plen) // 4 * 4)
            spec = P.SpecConfig(target_len=plen + 24, gamma1=2, gamma2=4, temperature=0.0, seed=i,
                                streaming=P.StreamingConfig(n_sink=2, budget=16),
                                retrieval=P.RetrievalConfig(chunk_size=4, budget=budget))
            out, _ = P.hierarchical_generate(tw, dw, prompt, spec)
            if out != ar:
                mismatches.append((i, frac))
    assert not mismatches, mismatches


def test_tensor_core_chunk_equals_steps_across_split_boundary(P):
    """head_dim 128 (tensor-core attention, fused RoPE + append): a 5-row
    decode_chunk whose appended slots straddle the 2,048-key split boundary
    is bit-identical to five decode_steps, and both match a prefill of the
    same tokens on the row-exact path."""
    from paper_2404_11912_b200 import model as M
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=128, d_ff=344, vocab_size=512, max_seq=2304)
    w = P.generate_weights(cfg, 23, tied_head=False)
    prompt = np.random.default_rng(8).integers(1, 512, 2046).tolist()
    tail = [5, 77, 301, 12, 450]
    a, b = P.FullCache.from_config(cfg), P.FullCache.from_config(cfg)
    P.prefill(w, prompt, a)
    P.prefill(w, prompt, b)
    rows = P.decode_chunk(w, tail, a)
    steps = np.stack([P.decode_step(w, tk, b) for tk in tail])
    assert np.array_equal(rows, steps)
    assert torch.equal(a.k[:, :, :2051], b.k[:, :, :2051]) and torch.equal(a.v[:, :, :2051], b.v[:, :, :2051])
    c = P.FullCache.from_config(cfg)
    ref = M._host_rows(M.forward_device(w, prompt + tail, c, None, prefill=False))[-5:]
    assert np.allclose(rows, ref, rtol=1e-4, atol=3e-4 * np.abs(ref).max())


def test_forward_randomized_configs_match_oracle(P):
    """Whole forwards on random geometries against the oracle (bf16 storage
    model): head_dim 64 / 128 (CUDA-core and tensor-core attention, fused
    RoPE), GQA ratios 1 / 2 / 4, prompts long enough for the GEMM prefill or
    not, then decode chunks crossing the 8-row block and single steps."""
    from oracle import hs_oracle as O
    rng = np.random.default_rng(77)
    for case in range(6):
        dh = int(rng.choice([64, 128]))
        kvh = int(rng.choice([1, 2, 4]))
        H = kvh * int(rng.choice([1, 2, 4]))
        cfg = P.ModelConfig(n_layers=2, n_heads=H, n_kv_heads=kvh, head_dim=dh, d_ff=int(rng.integers(3, 12)) * 32,
                            vocab_size=300, max_seq=1024)
        w = bf16_weights(P, P.generate_weights(cfg, 500 + case, tied_head=bool(case % 2)))
        om = O.OModel(O.OConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__}),
                      O.round_weights_bf16(w.tensors), w.tied_head)
        plen = int(rng.integers(20, 400))
        prompt = rng.integers(1, 300, plen).tolist()
        chunk = rng.integers(1, 300, int(rng.integers(2, 12))).tolist()
        steps = rng.integers(1, 300, 3).tolist()
        dc, oc = P.FullCache.from_config(cfg), O.OFullCache(2, kvh, dh, 1024, kv_bf16=True)
        got = [P.prefill(w, prompt, dc), P.decode_chunk(w, chunk, dc)]
        got += [P.decode_step(w, tk, dc)[None] for tk in steps]
        want = [O.prefill(om, prompt, oc), O.forward(om, chunk, oc)]
        oc.commit(oc.frontier)
        want += [O.decode_step(om, tk, oc)[None] for tk in steps]
        g, r = np.concatenate(got), np.concatenate(want)
        # fp32-accumulation differences in a K/V projection occasionally flip
        # the bf16 rounding of a cached entry (a 2^-8 step the oracle does
        # not share); over 2 layers that reaches ~3.4e-4 of the largest logit
        # (GEMM prefill, case 2) -- far inside the north star's 2e-2 bar
        assert np.allclose(g, r, rtol=1e-4, atol=1e-3 * np.abs(r).max()), (case, dh, H, kvh, plen)
        assert (np.argmax(g, -1) == np.argmax(r, -1)).mean() > 0.99, case


@pytest.mark.parametrize("case", range(4))
def test_randomized_sessions_match_oracle(P, case):
    """Random session geometries (target head_dim 64 / 128 -- the latter on
    the tensor-core attention with fused RoPE --, GQA, chunk / budget /
    stream sizes, gamma1 / gamma2, greedy and sampled) with planted models:
    token stream and per-level accept counts equal the oracle's exactly."""
    from oracle import hs_oracle as O
    rng = np.random.default_rng(300 + case)
    mk = lambda w: O.OModel(O.OConfig(**{k: getattr(w.config, k) for k in w.config.__dataclass_fields__}),
                            O.round_weights_bf16(w.tensors), w.tied_head)
    dh = [64, 128, 128, 64][case]
    kvh = int(rng.choice([1, 2]))
    tc = P.ModelConfig(n_layers=2, n_heads=kvh * 2, n_kv_heads=kvh, head_dim=dh, d_ff=192, vocab_size=400,
                       max_seq=1536)
    dc = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=32, d_ff=64, vocab_size=400, max_seq=1536)
    tw = bf16_weights(P, P.plant_successor(P.generate_weights(tc, 40 + case, tied_head=False), case, 0.85))
    dw = bf16_weights(P, P.plant_successor(P.generate_weights(dc, 50 + case, tied_head=False), case, 0.85))
    plen = int(rng.integers(100, 900))
    prompt = rng.integers(1, 400, plen).tolist()
    chunk = int(rng.choice([4, 8, 16]))
    budget = chunk * int(rng.integers(4, 24))
    stream = int(rng.choice([24, 48, 96]))
    g1, g2 = int(rng.integers(1, 4)), int(rng.integers(3, 7))
    temp = float([0.0, 0.6, 1.0, 0.6][case])
    spec = P.SpecConfig(target_len=plen + 40, gamma1=g1, gamma2=g2, temperature=temp, seed=case,
                        streaming=P.StreamingConfig(n_sink=4, budget=stream),
                        retrieval=P.RetrievalConfig(chunk_size=chunk, budget=budget, rebuild_stride=16))
    out, tr = P.HierarchicalSession(tw, dw, prompt, spec).generate()
    os_ = O.OSession(mk(tw), mk(dw), prompt, O.OSpec(target_len=plen + 40, gamma1=g1, gamma2=g2, temperature=temp,
                                                    seed=case, n_sink=4, stream_budget=stream, chunk=chunk,
                                                    retr_budget=budget, rebuild_stride=16), kv_bf16=True)
    oout, otr = os_.generate()
    assert out == oout, (case, dh, kvh, plen, chunk, budget, stream, g1, g2, temp)
    assert [tr.inner.proposed, tr.inner.accepted, tr.outer.proposed, tr.outer.accepted] == \
        [otr.inner[0], otr.inner[1], otr.outer[0], otr.outer[1]]
