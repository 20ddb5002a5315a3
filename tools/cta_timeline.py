#!/usr/bin/env python3
"""Per-CTA timeline of one lane forward (hs_cta_trace: globaltimer stamps
written by thread 0 of every CTA of the instrumented kernels), without a
profiler in the loop.  Reconstructs each kernel launch's span (first CTA
start -> last CTA end), the gaps between consecutive launches and the SM
coverage, so a forward's time splits into kernel time vs boundaries.

    HS_TRACE_BUILD=1 python paper_2404_11912_b200/build.py --force   # instrumented library
    python tools/cta_timeline.py [--lane retr|full|draft] [--t 3] [--ctx 16384]

(The instrumentation costs ~3% and is compiled out of the normal build.)
"""

from __future__ import annotations

import argparse
import collections
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

NAMES = {1: "gemv_tc", 2: "split_rows", 3: "norm_prep", 4: "attn_tc", 5: "attn_combine", 6: "embed", 7: "rope",
         8: "attn_partial"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lane", default="retr")
    ap.add_argument("--t", type=int, default=3)
    ap.add_argument("--ctx", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=8, help="layers shown in detail")
    ap.add_argument("--gemv", action="store_true",
                    help="per-GEMV CTA distributions (start = dependency release, griddepcontrol.wait)")
    ap.add_argument("--graph", action="store_true",
                    help="draft lane, t=1: replay the lane's captured step graph instead of a direct forward")
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200._abi import lib
    lib.hs_cta_trace.restype = C.c_int
    lib.hs_cta_trace.argtypes = [C.c_void_p, C.c_uint]
    tw = P.ModelWeights.on_device(P.DeviceModel.random(P.ModelConfig(**bench.TARGET_7B), 1))
    dw = P.ModelWeights.on_device(P.DeviceModel.random(P.ModelConfig(**bench.DRAFT_68M), 2))
    ctx = np.random.default_rng(0).integers(1, 32000, a.ctx).tolist()
    spec = P.SpecConfig(target_len=a.ctx + 64, gamma1=2, gamma2=4,
                        streaming=P.StreamingConfig(n_sink=4, budget=256),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
    lane = {"retr": sess.retr_lane, "full": sess.full_lane, "draft": sess.draft_lane}[a.lane]
    toks = torch.ones(a.t, dtype=torch.int32, device="cuda")
    f0 = lane.frontier
    fwd = (lambda: lane.step_graph_run(1)) if a.graph else (lambda: lane._forward(toks))
    for _ in range(3):
        fwd()
        lane.rollback_to(f0)
    cap = 1 << 18
    buf = torch.zeros(5 * cap * 3, dtype=torch.int64, device="cuda")   # 4 TU regions + GEMV phases
    torch.cuda.synchronize()
    lib.hs_cta_trace(buf.data_ptr(), cap)
    fwd()
    torch.cuda.synchronize()
    lib.hs_cta_trace(None, 0)
    lane.rollback_to(f0)
    rec = buf[:4 * cap * 3].view(-1, 3).cpu().numpy().astype(np.uint64)   # (region 5: GEMV phase records)
    rec = rec[rec[:, 1] > 0]
    kid_full = (rec[:, 0] >> np.uint64(32)).astype(int)
    kid = kid_full & 0xff
    t0 = rec[:, 1].astype(np.int64)
    t1 = rec[:, 2].astype(np.int64)
    base = t0.min()
    t0 -= base
    t1 -= base
    # group CTAs into launches: same kernel id, ordered by start; a new launch starts when
    # a CTA of the same kernel starts after every earlier CTA of that launch ended + a gap
    order = np.argsort(t0, kind="stable")
    launches = []
    for i in order:
        k = kid[i]
        cur = launches[-1] if launches and launches[-1]["kid"] == k else None
        if cur is not None and t0[i] <= cur["end"] + 500:
            cur["start"] = min(cur["start"], t0[i])
            cur["end"] = max(cur["end"], t1[i])
            cur["ctas"] += 1
            cur["busy"] += t1[i] - t0[i]
        else:
            launches.append({"kid": k, "start": t0[i], "end": t1[i], "ctas": 1, "busy": t1[i] - t0[i]})
    span = max(l["end"] for l in launches)
    if a.gemv:
        gemv_tails(kid_full, t0, t1, a.layers)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    prev_end = 0
    gaps = 0.0
    for l in launches:
        g = max(0, l["start"] - prev_end)
        gaps += g
        a_ = agg[NAMES[l["kid"]]]
        a_[0] += 1
        a_[1] += (l["end"] - l["start"]) / 1e3
        a_[2] += g / 1e3
        prev_end = max(prev_end, l["end"])
    print(f"lane {a.lane} t={a.t}: span {span / 1e3:.1f} us, {len(launches)} launches, gaps {gaps / 1e3:.1f} us")
    for n, (c, d, g) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {n:14s} x{c:4d}  span {d:9.1f} us ({d / c:7.2f} avg)  gap-before {g:8.1f} us ({g / c:5.2f} avg)")
    print("first launches (start, span, ctas, mean CTA time, us):")
    for l in launches[:12 * a.layers // 8 + 12]:
        print(f"  {NAMES[l['kid']]:14s} {l['start'] / 1e3:9.2f} {(l['end'] - l['start']) / 1e3:8.2f} {l['ctas']:5d} "
              f"{l['busy'] / l['ctas'] / 1e3:7.2f}")


def gemv_tails(kid_full, t0, t1, layers):
    """Launches (GEMVs carry their tile count in bits 8+ of the id): per launch the CTA
    release times (after griddepcontrol.wait) and end times, relative to the
    first release, and the idle time until the next GEMV's first release."""
    sel = np.arange(len(kid_full))
    order = sel[np.argsort(t0[sel], kind="stable")]
    groups, cur = [], None
    for i in order:
        if cur is None or kid_full[i] != cur[0]:
            cur = (kid_full[i], [])
            groups.append(cur)
        cur[1].append(i)
    print("launches: kernel [gemv tiles] ctas | release spread | end p10 p50 p90 max (us from first release) | "
          "next release")
    for j, (k, idx) in enumerate(groups[:8 * layers + 4]):
        idx = np.array(idx)
        r0 = t0[idx].min()
        rel = (t0[idx] - r0) / 1e3
        end = (t1[idx] - r0) / 1e3
        nxt = (t0[np.array(groups[j + 1][1])].min() - r0) / 1e3 if j + 1 < len(groups) else float("nan")
        print(f"  {NAMES[k & 0xff]:12s} {k >> 8:4d} {len(idx):5d} | {rel.max():6.2f} | {np.percentile(end, 10):6.2f} {np.median(end):6.2f} "
              f"{np.percentile(end, 90):6.2f} {end.max():6.2f} | {nxt:7.2f}")


if __name__ == "__main__":
    main()
