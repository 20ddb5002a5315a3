"""Pin the CPU oracle to the reference: every golden fixture produced by
`tests/golden/make_golden.py` (which ran the reference package in place) is
reproduced bit-for-bit by `oracle/hs_oracle.py`.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import hs_oracle as O
from tests.conftest import small_cfg


def _model(cfg, seed, tied, mode):
    t = O.make_tensors(cfg, seed, tied)
    if mode == "bf16":
        t = O.round_weights_bf16(t)
    return O.OModel(cfg, t, tied)


def test_score_chunks_bitwise(golden):
    data, meta = golden
    for i, c in enumerate(meta["score_cases"]):
        r = np.random.default_rng(c["seed"])
        keys = r.normal(0, 1, (c["L"], c["kvh"], c["dh"])).astype(np.float32)
        q = r.normal(0, 1, (c["kvh"] * c["g"], c["dh"])).astype(np.float32)
        b, s = O.chunk_scores(keys, q, c["chunk"], c["kvh"])
        assert np.array_equal(b, data[f"score/{i}/bounds"])
        assert np.array_equal(s, data[f"score/{i}/scores"]), f"case {i}"


def test_build_and_overwrite(golden):
    data, meta = golden
    for i, c in enumerate(meta["build_cases"]):
        r = np.random.default_rng(c["seed"])
        src = O.OFullCache(c["layers"], c["kvh"], c["dh"], 4096)
        for li in range(c["layers"]):
            k = r.normal(0, 1, (c["L"], c["kvh"], c["dh"])).astype(np.float32)
            src.append(li, k, -k)
        src.commit(c["L"])
        qs = [r.normal(0, 1, (c["H"], c["dh"])).astype(np.float32) for _ in range(c["layers"])]
        rc = O.ORetrievalCache(c["layers"], c["kvh"], c["dh"], c["chunk"], c["budget"])
        (tab, clamped) = rc.build(src, qs, c["L"])
        assert int(clamped) == int(data[f"build/{i}/clamped"])
        for li in range(c["layers"]):
            assert tab[li][2] == data[f"build/{i}/selected/{li}"].tolist()
            assert np.array_equal(rc.positions(li), data[f"build/{i}/exposed0/{li}"])
            assert rc.victims[li] == data[f"build/{i}/victims/{li}"].tolist()
        for step in range(5):
            for li in range(c["layers"]):
                k = np.full((1, c["kvh"], c["dh"]), float(c["L"] + step), np.float32)
                rc.append(li, k, -k)
            rc.commit(c["L"] + step + 1)
        for li in range(c["layers"]):
            k = np.full((3, c["kvh"], c["dh"]), 0.5, np.float32)
            rc.append(li, k, -k)
        rc.commit(c["L"] + 8)
        for li in range(c["layers"]):
            assert np.array_equal(rc.positions(li), data[f"build/{i}/exposed1/{li}"])


@pytest.mark.parametrize("mode", ["plain", "bf16"])
def test_forward_bitwise(golden, mode):
    data, meta = golden
    for c in meta["forward_cases"]:
        cfg = O.OConfig(**c["cfg"])
        m = _model(cfg, c["seed"], c["tied"], mode)
        cache = O.OFullCache(cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, cfg.max_seq,
                             kv_bf16=(mode == "bf16"))
        rec = O.ORecorder()
        lg = O.prefill(m, c["prefill"], cache, rec)
        name = c["name"]
        assert np.array_equal(lg, data[f"fwd/{name}/{mode}/prefill"]), name
        assert np.array_equal(np.stack(rec.last_queries), data[f"fwd/{name}/{mode}/q_last"])
        rows = [O.decode_step(m, tk, cache) for tk in c["decode"]]
        assert np.array_equal(np.stack(rows), data[f"fwd/{name}/{mode}/decode"]), name


def test_verify_and_correct(golden):
    data, meta = golden
    for i, c in enumerate(meta["verify_cases"]):
        q, p, x = data[f"verify/{i}/q"], data[f"verify/{i}/p"], data[f"verify/{i}/x"]
        r = np.random.default_rng(c["rng_seed"])
        acc = [int(O.accept(int(xx), q, p, r)) for xx in x]
        cor = [O.resample(q, p, r) for _ in range(20)]
        assert acc == data[f"verify/{i}/acc"].tolist()
        assert cor == data[f"verify/{i}/cor"].tolist()


def test_autoregressive(golden):
    data, meta = golden
    for i, c in enumerate(meta["ar_cases"]):
        m = _model(small_cfg(), c["seed"], True, "plain")
        out = O.ar_generate(m, [1, 2, 3], 14, c["temperature"], seed=c["rng_seed"])
        assert out == data[f"ar/{i}/tokens"].tolist()


def _small_session(kw, mode):
    kw = dict(kw)
    cfg = small_cfg()
    target = _model(cfg, 11, True, mode)
    draft = _model(small_cfg(n_layers=1), 12, True, mode)
    prefix_len = kw.pop("prefix_len", 24)
    rng = np.random.default_rng(99)
    prefix = rng.integers(1, cfg.vocab_size, prefix_len).tolist()
    spec = O.OSpec(target_len=kw.pop("target_len", prefix_len + 12), gamma1=kw.pop("gamma1", 2),
                   gamma2=kw.pop("gamma2", 4), temperature=kw.pop("temperature", 0.0), seed=5,
                   n_sink=2, stream_budget=12, chunk=kw.pop("chunk", 4), retr_budget=kw.pop("budget", 16),
                   rebuild_stride=kw.pop("rebuild_stride", 128),
                   rolling_window=kw.pop("rolling_window", 16))
    assert not kw
    return O.OSession(target, draft, prefix, spec, kv_bf16=(mode == "bf16"))


def _check_trace(data, tag, out, tr):
    assert out == data[tag + "/tokens"].tolist()
    s = tr.summary()
    assert [s["inner"]["proposed"], s["inner"]["accepted"], s["inner"]["rounds"],
            s["outer"]["proposed"], s["outer"]["accepted"], s["outer"]["rounds"]] == \
        data[tag + "/stats"].tolist()
    levels = ["draft", "retrieval", "corrected", "bonus"]
    assert [levels.index(r["level"]) for r in tr.records] == data[tag + "/rec_level"].tolist()
    assert [r["outer_round"] for r in tr.records] == data[tag + "/rec_round"].tolist()


@pytest.mark.parametrize("mode", ["plain", "bf16"])
def test_small_sessions(golden, mode):
    data, meta = golden
    for i, kw in enumerate(meta["small_sessions"]):
        out, tr = _small_session(kw, mode).generate()
        _check_trace(data, f"sess/{i}/{mode}", out, tr)


@pytest.mark.slow
def test_cfg1_sessions(golden):
    """BASELINE config 1 (4K context) -- the oracle reproduces the reference's
    greedy and T=0.6 streams, traces and initial top-k selections."""
    data, meta = golden
    c = meta["cfg1"]
    tcfg, dcfg = O.OConfig(**c["target"]), O.OConfig(**c["draft"])
    prompt = np.random.default_rng(0).integers(1, 256, 4096).tolist()
    for mode, temp in [("plain", 0.0), ("bf16", 0.6)]:
        t = _model(tcfg, 1, False, mode)
        d = _model(dcfg, 2, False, mode)
        spec = O.OSpec(target_len=4096 + 64, gamma1=2, gamma2=4, temperature=temp, seed=0,
                       n_sink=4, stream_budget=256, chunk=8, retr_budget=256)
        sess = O.OSession(t, d, prompt, spec, kv_bf16=(mode == "bf16"))
        tag = f"cfg1/{mode}/T{temp}"
        imp0 = [row[2] for row in sess.builds[0][0]]
        assert imp0 == data[tag + "/importance0"].tolist()
        out, tr = sess.generate()
        assert out[4096:] == data[tag + "/tokens"].tolist()
        s = tr.summary()
        assert [s["inner"]["proposed"], s["inner"]["accepted"], s["inner"]["rounds"],
                s["outer"]["proposed"], s["outer"]["accepted"], s["outer"]["rounds"]] == \
            data[tag + "/stats"].tolist()


def test_shard_merge_matches_unsharded():
    """Sequence-sharding model (§8(e)): merging per-shard partial softmax
    states equals unsharded attention."""
    rng = np.random.default_rng(0)
    q = rng.normal(0, 1, (5, 16))
    K = rng.normal(0, 1, (300, 16))
    V = rng.normal(0, 1, (300, 16))
    scale = 0.25
    s = q @ K.T * scale
    p = np.exp(s - s.max(axis=1, keepdims=True))
    ref = (p / p.sum(axis=1, keepdims=True)) @ V
    for bounds in ([0, 300], [0, 100, 300], [0, 64, 128, 192, 300], [0, 0, 150, 300]):
        got = O.merge_partials(O.shard_partials(q, K, V, bounds, scale))
        assert np.allclose(got, ref, atol=1e-12)
