#!/usr/bin/env python3
"""BASELINE config 5: retrieval-budget / chunk-size sweep at a 256K context
(Llama2-7B shape, one B200): for every (budget, chunk) point the same full
cache is reused, the retrieval lane is rebuilt with that configuration, and
`generate()` runs for --tokens tokens.  Reports ms/token, acceptance rates,
the per-token algorithmic bytes and the achieved HBM GB/s (all forwards and
builds / device time), plus the build cost.

    python tools/sweep.py [--context 262144] [--tokens 64] [--json out.json]

Synthetic state (random N(0,1) K/V, planted-successor weights; bench.py):
the acceptance rates therefore reflect the planted channel, not a real
model's attention locality -- the point of the sweep is cost vs budget/chunk.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=262144)
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--budgets", type=int, nargs="+", default=[1024, 2048, 4096, 8192, 16384])
    ap.add_argument("--chunks", type=int, nargs="+", default=[8, 16, 32])
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200 import speculation as S
    from paper_2404_11912_b200.runtime import STATS
    tshape = {**bench.TARGET_7B, "max_seq": a.context + 4096}
    tdm = P.DeviceModel.random(P.ModelConfig(**tshape), 1)
    ddm = P.DeviceModel.random(P.ModelConfig(**{**bench.DRAFT_68M, "max_seq": a.context + 4096}), 1001)
    tdm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    ddm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    tw, dw = P.ModelWeights.on_device(tdm), P.ModelWeights.on_device(ddm)
    ctx = np.random.default_rng(0).integers(1, 32000, a.context).tolist()
    spec = P.SpecConfig(target_len=a.context + 1, gamma1=bench.GAMMA1, gamma2=bench.GAMMA2,
                        streaming=P.StreamingConfig(n_sink=bench.SINK, budget=bench.STREAM),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
    base_committed = list(sess.committed)
    full_f, full_c = sess.full_lane.cache.frontier, sess.full_lane.cache.committed
    draft_state = sess.draft_lane.clone()
    rows = []
    for budget in a.budgets:
        for chunk in a.chunks:
            # fresh lanes over the same full cache and draft state
            sess.committed = list(base_committed)
            sess.full_lane.rollback_to(full_f)
            sess.full_lane.cache.committed = full_c
            sess.full_lane.frontier_logits = None
            sess.draft_lane = draft_state.clone()
            sess.config.retrieval = P.RetrievalConfig(chunk_size=chunk, budget=budget)
            sess.retr_lane = S.Lane(tw, P.RetrievalCache.from_config(tw.config, sess.config.retrieval))
            sess.rolling = P.RollingAcceptance(sess.config.retrieval.rolling_window)
            sess.tokens_since_build = 0
            # the full lane re-decodes the last committed token for its logits and the build query
            sess.full_lane.rollback_to(full_f - 1)
            sess.full_lane.cache.committed = full_f - 1
            sess.full_lane.advance([base_committed[-1]])
            sess.full_lane.commit()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sess._initial_build()
            e1.record()
            torch.cuda.synchronize()
            build_ms = e0.elapsed_time(e1)
            sess.config.target_len = len(sess.committed) + 8          # warm-up
            sess.generate(seed=1)
            c0 = dict(S.COUNTERS)
            b0 = STATS["alg_bytes"]
            n0 = len(sess.committed)
            sess.config.target_len = n0 + a.tokens
            torch.cuda.synchronize()
            e0.record()
            sess.generate(seed=2)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            got = len(sess.committed) - n0
            d = {k: S.COUNTERS[k] - c0.get(k, 0) for k in S.COUNTERS}
            alg = STATS["alg_bytes"] - b0
            row = {"budget": budget, "chunk": chunk, "ms_per_token": ms / got,
                   "inner_rate": d["inner_accepted"] / max(1, d["inner_proposed"]),
                   "outer_rate": d["outer_accepted"] / max(1, d["outer_proposed"]),
                   "alg_GB_per_token": alg / got / 1e9, "achieved_GBps": alg / (ms / 1e3) / 1e9,
                   "build_ms": build_ms, "rebuilds": d["rebuilds"]}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"context": a.context, "tokens": a.tokens, "points": rows}, f, indent=1)


if __name__ == "__main__":
    main()
