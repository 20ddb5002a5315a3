#!/usr/bin/env python3
"""Where one TriForce decode step spends its time (torch.profiler / CUPTI):
GPU busy time per kernel family, and the idle time between kernels (host
work, syncs, launch latency), for a `generate()` call that commits --gen
tokens at the Llama2-7B shape.

    python tools/round_timeline.py [--ctx 32768] [--gen 16]
"""

from __future__ import annotations

import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--gen", type=int, default=16)
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    tdm, ddm = P.DeviceModel.random(P.ModelConfig(**bench.TARGET_7B), seed=1), \
        P.DeviceModel.random(P.ModelConfig(**bench.DRAFT_68M), seed=1001)
    tdm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    ddm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    tw, dw = P.ModelWeights.on_device(tdm), P.ModelWeights.on_device(ddm)
    ctx = np.random.default_rng(0).integers(1, 32000, a.ctx).tolist()
    spec = P.SpecConfig(target_len=a.ctx + 1, gamma1=2, gamma2=4,
                        streaming=P.StreamingConfig(n_sink=4, budget=256),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
    for i in range(3):
        sess.config.target_len = len(sess.committed) + a.gen
        sess.generate(seed=i)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    sess.config.target_len = len(sess.committed) + a.gen
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        sess.generate(seed=99)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
    t0, t1 = ks[0][0], max(e for _, e, _ in ks)
    busy = collections.Counter()
    count = collections.Counter()
    idle = 0.0
    end = t0
    gaps = []
    prev = "start"
    for s, e, n in ks:
        if s > end:
            gaps.append((s - end, prev, n.split("(")[0][:40], (s - t0) / 1e3))
        prev = n.split("(")[0][:40]
        name = n.split("(")[0].split("<")[0].replace("hs::", "").replace("(anonymous namespace)::", "").strip()
        name = name or "attn_tc_kernel"
        busy[name] += e - s
        count[name] += 1
        if s > end:
            idle += s - end
        end = max(end, e)
    span = t1 - t0
    print(f"generate({a.gen} tokens) at ctx {a.ctx}: span {span / 1e3:.2f} ms, GPU idle {idle / 1e3:.2f} ms "
          f"({100 * idle / span:.1f}%), {len(ks)} kernels")
    for n, v in busy.most_common(25):
        print(f"  {v / 1e3:8.3f} ms  {count[n]:6d} x  {n}")
    gaps.sort(reverse=True)
    big = [g for g in gaps if g[0] > 20]
    print(f"idle gaps > 20 us: {len(big)}, total {sum(g[0] for g in big) / 1e3:.2f} ms; largest:")
    for g, a_, b_, at in gaps[:25]:
        print(f"  {g:8.1f} us at {at:8.2f} ms  after {a_:40s} before {b_}")
    # idle time by (previous op -> next op) pair
    pairs = collections.defaultdict(lambda: [0, 0.0])
    short = lambda n: n.replace("hs::", "").replace("void ", "").replace("(anonymous namespace)::", "").split("<")[0][:28]
    for g, a_, b_, at in gaps:
        k = (short(a_), short(b_))
        pairs[k][0] += 1
        pairs[k][1] += g
    print("idle by (after -> before), all gaps:")
    for (a_, b_), (c, g) in sorted(pairs.items(), key=lambda x: -x[1][1])[:25]:
        print(f"  {g / 1e3:8.3f} ms  {c:6d} x  {g / c:7.1f} us  {a_:28s} -> {b_}")


if __name__ == "__main__":
    main()
