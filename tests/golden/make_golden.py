"""Generate golden fixtures by running the REFERENCE package in place.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `hierspec` from /root/reference/pkg/src (read-only, unmodified)
and writes `tests/golden/ref_golden.npz` + `tests/golden/ref_golden.json`.
The GPU box has no /root/reference; tests there read only these files.

Two families of fixtures:
  * plain reference behaviour (pins oracle/hs_oracle.py bit-for-bit);
  * "bf16 storage" behaviour: the reference run with bf16-rounded weight
    matrices and with caches whose `append` rounds K/V rows to bf16 (a
    test-side subclass).  This is the GPU storage model,
    so GPU parity tests compare against these directly.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import hierspec  # noqa: E402
import hierspec.speculation as hspec  # noqa: E402
from hierspec.caches import (FullCache, RetrievalCache, RetrievalConfig,  # noqa: E402
                             StreamingCache, StreamingConfig, score_chunks)
from hierspec.model import (ForwardRecorder, ModelConfig, ModelWeights,  # noqa: E402
                            decode_step, generate_weights, prefill)
from hierspec.speculation import (HierarchicalSession, SpecConfig,  # noqa: E402
                                  autoregressive_generate, correct_token,
                                  verify_token)

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = {}
META = {}


def bf16(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


def bf16_weights(w: ModelWeights) -> ModelWeights:
    t = {n: (x.copy() if "norm" in n else bf16(x)) for n, x in w.tensors.items()}
    return ModelWeights(w.config, t, w.tied_head).validate()


class _Round:
    def append(self, layer, k, v):
        return super().append(layer, bf16(k), bf16(v))


class RFull(_Round, FullCache):
    pass


class RStream(_Round, StreamingCache):
    pass


class RRetr(_Round, RetrievalCache):
    pass


class bf16_caches:
    """Context manager swapping the session's cache classes for rounding ones."""

    def __enter__(self):
        self.saved = (hspec.FullCache, hspec.StreamingCache, hspec.RetrievalCache)
        hspec.FullCache, hspec.StreamingCache, hspec.RetrievalCache = RFull, RStream, RRetr

    def __exit__(self, *a):
        hspec.FullCache, hspec.StreamingCache, hspec.RetrievalCache = self.saved


def small_config(**kw):
    base = dict(n_layers=2, n_heads=4, n_kv_heads=4, head_dim=8, d_ff=32,
                vocab_size=40, max_seq=128, rope_theta=10000.0, norm_eps=1e-5)
    base.update(kw)
    return ModelConfig(**base)


def cfg1_target():
    return ModelConfig(n_layers=2, n_heads=4, n_kv_heads=4, head_dim=64, d_ff=688,
                       vocab_size=260, max_seq=4224)


def cfg1_draft():
    return ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=64, d_ff=344,
                       vocab_size=260, max_seq=4224)


def put(name, arr):
    OUT[name] = np.asarray(arr)


# ---------------------------------------------------------------------------
def gen_score_chunks():
    cases = []
    rng = np.random.default_rng(42)
    for i in range(24):
        L = int(rng.integers(9, 300))
        kvh = int(rng.choice([1, 2, 4]))
        g = int(rng.choice([1, 2]))
        dh = int(rng.choice([4, 8, 64, 128]))
        chunk = int(rng.choice([1, 4, 8, 16, 32]))
        seed = 1000 + i
        r = np.random.default_rng(seed)
        keys = r.normal(0, 1, (L, kvh, dh)).astype(np.float32)
        q = r.normal(0, 1, (kvh * g, dh)).astype(np.float32)
        b, s = score_chunks(keys, q, chunk, kvh)
        put(f"score/{i}/bounds", b)
        put(f"score/{i}/scores", s)
        cases.append(dict(L=L, kvh=kvh, g=g, dh=dh, chunk=chunk, seed=seed))
    META["score_cases"] = cases


def gen_build():
    """RetrievalCache.build + overwrite sequence on random sources."""
    cases = []
    for i, (L, chunk, budget, layers, kvh, dh, H) in enumerate([
            (64, 4, 16, 2, 2, 8, 4), (100, 8, 32, 2, 2, 16, 4), (37, 4, 8, 1, 1, 8, 2),
            (16, 4, 16, 2, 2, 4, 2), (300, 16, 64, 3, 4, 32, 8), (129, 8, 128, 2, 2, 8, 4)]):
        seed = 7000 + i
        r = np.random.default_rng(seed)
        src = FullCache(layers, kvh, dh, 4096)
        for li in range(layers):
            k = r.normal(0, 1, (L, kvh, dh)).astype(np.float32)
            src.append(li, k, -k)
        src.commit(L)
        qs = [r.normal(0, 1, (H, dh)).astype(np.float32) for _ in range(layers)]
        rc = RetrievalCache(layers, kvh, dh, RetrievalConfig(chunk_size=chunk, budget=budget))
        tab = rc.build(src, qs, upto=L)
        for li in range(layers):
            put(f"build/{i}/selected/{li}", np.array(tab.selected[li]))
            put(f"build/{i}/exposed0/{li}", rc.exposed_positions(li))
            put(f"build/{i}/victims/{li}", np.array(rc._victims[li]))
        # commit 5 new positions one at a time and 3 at once
        for step in range(5):
            for li in range(layers):
                k = np.full((1, kvh, dh), float(L + step), np.float32)
                rc.append(li, k, -k)
            rc.commit(L + step + 1)
        for li in range(layers):
            k = np.full((3, kvh, dh), 0.5, np.float32)
            rc.append(li, k, -k)
        rc.commit(L + 8)
        for li in range(layers):
            put(f"build/{i}/exposed1/{li}", rc.exposed_positions(li))
        put(f"build/{i}/clamped", np.array(int(tab.clamped)))
        cases.append(dict(L=L, chunk=chunk, budget=budget, layers=layers, kvh=kvh, dh=dh, H=H, seed=seed))
    META["build_cases"] = cases


def gen_forward():
    # prefill + decode logits for three configurations, plain and bf16
    specs = [("small", small_config(), 11, True, [1, 5, 9, 3, 22, 17, 8], [9, 10, 11]),
             ("gqa", small_config(n_kv_heads=2), 4, True, [1, 2, 3, 4, 5, 6], [7, 1]),
             ("untied", small_config(n_layers=3, head_dim=16, d_ff=48, vocab_size=64), 5, False,
              list(range(1, 30)), [3, 4, 5, 6])]
    META["forward_cases"] = []
    for name, cfg, seed, tied, toks, dec in specs:
        for mode in ("plain", "bf16"):
            w = generate_weights(cfg, seed, tied)
            if mode == "bf16":
                w = bf16_weights(w)
                cache = RFull.from_config(cfg)
            else:
                cache = FullCache.from_config(cfg)
            rec = ForwardRecorder()
            lg = prefill(w, toks, cache, rec)
            put(f"fwd/{name}/{mode}/prefill", lg)
            put(f"fwd/{name}/{mode}/q_last", np.stack(rec.last_queries))
            rows = [decode_step(w, tk, cache) for tk in dec]
            put(f"fwd/{name}/{mode}/decode", np.stack(rows))
        META["forward_cases"].append(dict(name=name, cfg=cfg.__dict__, seed=seed, tied=tied,
                                          prefill=toks, decode=dec))


def trace_arrays(prefix, tr):
    recs = tr.records
    put(prefix + "/rec_tok", np.array([r["token"] for r in recs]))
    put(prefix + "/rec_level", np.array([["draft", "retrieval", "corrected", "bonus"].index(r["level"])
                                         for r in recs]))
    put(prefix + "/rec_acc", np.array([int(r["accepted"]) for r in recs]))
    put(prefix + "/rec_round", np.array([r["outer_round"] for r in recs]))
    s = tr.summary()
    put(prefix + "/stats", np.array([s["inner"]["proposed"], s["inner"]["accepted"], s["inner"]["rounds"],
                                     s["outer"]["proposed"], s["outer"]["accepted"], s["outer"]["rounds"]]))


def gen_small_sessions():
    """The reference's own build_session fixture (tests/test_speculation.py:89-104)."""
    cases = []

    def build(seed_t=11, seed_d=12, prefix_len=24, target_len=None, temperature=0.0, gamma1=2,
              gamma2=4, budget=16, chunk=4, stream_budget=12, **over):
        cfg = small_config()
        target = generate_weights(cfg, seed_t)
        draft = generate_weights(small_config(n_layers=1), seed_d)
        rng = np.random.default_rng(99)
        prefix = rng.integers(1, cfg.vocab_size, prefix_len).tolist()
        spec = SpecConfig(target_len=target_len or prefix_len + 12, gamma1=gamma1, gamma2=gamma2,
                          temperature=temperature, seed=5,
                          streaming=StreamingConfig(n_sink=2, budget=stream_budget),
                          retrieval=RetrievalConfig(chunk_size=chunk, budget=budget, **over))
        return target, draft, prefix, spec

    plan = [dict(budget=8, chunk=4, prefix_len=20, target_len=36),
            dict(budget=16, chunk=4, prefix_len=20, target_len=36),
            dict(budget=32, chunk=4, prefix_len=20, target_len=36),
            dict(temperature=1.0, target_len=40),
            dict(temperature=0.7, target_len=44),
            dict(budget=8, chunk=4, prefix_len=20, target_len=44, rebuild_stride=6, rolling_window=4),
            dict(temperature=0.6, target_len=48, rebuild_stride=8, rolling_window=3),
            dict(temperature=0.5, target_len=40, gamma1=3, gamma2=5)]
    for i, kw in enumerate(plan):
        for mode in ("plain", "bf16"):
            target, draft, prefix, spec = build(**kw)
            if mode == "bf16":
                target, draft = bf16_weights(target), bf16_weights(draft)
                with bf16_caches():
                    out, tr = HierarchicalSession(target, draft, prefix, spec).generate()
            else:
                out, tr = HierarchicalSession(target, draft, prefix, spec).generate()
            put(f"sess/{i}/{mode}/tokens", np.array(out))
            trace_arrays(f"sess/{i}/{mode}", tr)
        cases.append(kw)
    META["small_sessions"] = cases


def gen_ar():
    cases = []
    for i, (seed, temp, s2) in enumerate([(3, 0.9, 4), (3, 0.0, 4), (5, 0.5, 0), (7, 1.0, 11)]):
        cfg = small_config()
        w = generate_weights(cfg, seed)
        out = autoregressive_generate(w, [1, 2, 3], 14, temp, seed=s2)
        put(f"ar/{i}/tokens", np.array(out))
        cases.append(dict(seed=seed, temperature=temp, rng_seed=s2))
    META["ar_cases"] = cases


def gen_verify():
    rng = np.random.default_rng(3)
    cases = []
    for i in range(6):
        V = int(rng.integers(3, 40))
        q = rng.dirichlet(np.ones(V))
        p = rng.dirichlet(np.ones(V) * 0.5)
        x = [int(rng.integers(0, V)) for _ in range(20)]
        r = np.random.default_rng(100 + i)
        acc = [int(verify_token(xx, q, p, r)) for xx in x]
        cor = [correct_token(q, p, r) for _ in range(20)]
        put(f"verify/{i}/q", q)
        put(f"verify/{i}/p", p)
        put(f"verify/{i}/x", np.array(x))
        put(f"verify/{i}/acc", np.array(acc))
        put(f"verify/{i}/cor", np.array(cor))
        cases.append(dict(V=V, rng_seed=100 + i))
    META["verify_cases"] = cases


def gen_cfg1():
    """BASELINE config 1 at 4K context: tiny untied Llama, chunk 8, budget 256."""
    tw = generate_weights(cfg1_target(), 1, tied_head=False)
    dw = generate_weights(cfg1_draft(), 2, tied_head=False)
    prompt = np.random.default_rng(0).integers(1, 256, 4096).tolist()
    META["cfg1"] = dict(target=cfg1_target().__dict__, draft=cfg1_draft().__dict__, target_seed=1,
                        draft_seed=2, prompt_seed=0, prompt_len=4096, gen=64, chunk=8, budget=256,
                        n_sink=4, stream_budget=256, gamma1=2, gamma2=4)
    runs = [("plain", 0.0), ("bf16", 0.0), ("bf16", 0.6)]
    for mode, temp in runs:
        t, d = (tw, dw) if mode == "plain" else (bf16_weights(tw), bf16_weights(dw))
        spec = SpecConfig(target_len=4096 + 64, gamma1=2, gamma2=4, temperature=temp, seed=0,
                          streaming=StreamingConfig(n_sink=4, budget=256),
                          retrieval=RetrievalConfig(chunk_size=8, budget=256))
        tag = f"cfg1/{mode}/T{temp}"
        if mode == "bf16":
            with bf16_caches():
                sess = HierarchicalSession(t, d, prompt, spec)
                imp0 = [list(x) for x in sess.retr_lane.cache.table.selected]
                sc0 = np.stack(sess.retr_lane.cache.table.scores)
                out, tr = sess.generate()
        else:
            sess = HierarchicalSession(t, d, prompt, spec)
            imp0 = [list(x) for x in sess.retr_lane.cache.table.selected]
            sc0 = np.stack(sess.retr_lane.cache.table.scores)
            out, tr = sess.generate()
        put(tag + "/tokens", np.array(out[4096:]))
        put(tag + "/importance0", np.array(imp0))
        put(tag + "/scores0", sc0)   # the initial build's fp64 chunk scores per layer (near-tie analysis)
        trace_arrays(tag, tr)
        print(tag, tr.summary(), flush=True)
    # AR greedy with bf16 storage for the GPU AR parity test
    with bf16_caches():
        w = bf16_weights(tw)
        c = hspec.FullCache.from_config(w.config)
        rec = ForwardRecorder()
        lg = prefill(w, prompt, c, rec)
        put("cfg1/bf16/prefill_last", lg[-1])
        put("cfg1/bf16/q_last", np.stack(rec.last_queries))


def main():
    gen_score_chunks()
    gen_build()
    gen_forward()
    gen_verify()
    gen_ar()
    gen_small_sessions()
    gen_cfg1()
    np.savez_compressed(os.path.join(HERE, "ref_golden.npz"), **OUT)
    META["reference_version"] = hierspec.__version__
    META["numpy"] = np.__version__
    with open(os.path.join(HERE, "ref_golden.json"), "w") as f:
        json.dump(META, f, indent=1, sort_keys=True)
    print("wrote", len(OUT), "arrays")


if __name__ == "__main__":
    main()
