#!/usr/bin/env python3
"""Kernel timeline of single lane forwards (torch.profiler / CUPTI): per
kernel start, duration and the idle gap before it, to see where a forward
loses time to launch gaps versus kernel time.

    python tools/timeline.py [--ctx 16384] [--t 3] [--lane retr|full|draft]
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=16384)
    ap.add_argument("--t", type=int, default=3)
    ap.add_argument("--lane", default="retr")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    import paper_2404_11912_b200 as P
    import bench
    tcfg = P.ModelConfig(**{**bench.TARGET_7B, "n_layers": a.layers})
    dcfg = P.ModelConfig(**bench.DRAFT_68M)
    tw = P.ModelWeights.on_device(P.DeviceModel.random(tcfg, seed=1))
    dw = P.ModelWeights.on_device(P.DeviceModel.random(dcfg, seed=2))
    ctx = np.random.default_rng(0).integers(1, 32000, a.ctx).tolist()
    spec = P.SpecConfig(target_len=a.ctx + 64, gamma1=2, gamma2=4,
                        streaming=P.StreamingConfig(n_sink=4, budget=256),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
    lane = {"retr": sess.retr_lane, "full": sess.full_lane, "draft": sess.draft_lane}[a.lane]
    toks = torch.ones(a.t, dtype=torch.int32, device="cuda")
    f0 = lane.frontier
    for _ in range(3):
        lane._forward(toks)
        lane.rollback_to(f0)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        lane._forward(toks)
        torch.cuda.synchronize()
    lane.rollback_to(f0)
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
    t0 = ks[0][0]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    prev_end = t0
    for s, e, n in ks:
        name = n.split("(")[0].split("<")[0].replace("hs::", "").replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += e - s
        agg[name][2] += max(0.0, s - prev_end)
        prev_end = max(prev_end, e)
    total = ks[-1][1] - t0
    busy = sum(v[1] for v in agg.values())
    print(f"lane={a.lane} t={a.t} layers={a.layers}: span {total:.1f} us, kernel time {busy:.1f} us, "
          f"gaps {sum(v[2] for v in agg.values()):.1f} us, {len(ks)} kernels")
    for n, (c, d, g) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c:5d} x {n:40s} {d:9.1f} us ({d / c:7.2f} avg)  gaps-before {g:8.1f} us")
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"span_us": total, "busy_us": busy, "kernels": {k: v for k, v in agg.items()}}, f, indent=1)


if __name__ == "__main__":
    main()
