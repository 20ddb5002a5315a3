#!/usr/bin/env python3
"""Per-CTA phase breakdown of every GEMV in one lane forward (trace build only:
HS_TRACE_BUILD=1 python paper_2404_11912_b200/build.py --force).  Each GEMV CTA
stamps start, dependency release, first / last weight stage landed (seen by
the MMA thread), accumulator complete, split-K reduction + epilogue done, end.
Prints, per GEMV kind (tile count x split), medians over layers of the launch's
phases relative to its first release.

    python tools/gemv_phases.py [--lane retr] [--t 3] [--ctx 16384]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lane", default="retr")
    ap.add_argument("--t", type=int, default=3)
    ap.add_argument("--ctx", type=int, default=16384)
    ap.add_argument("--raw", default=None, help="also save the raw [n][16] records (.npy)")
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
    for _ in range(3):
        lane._forward(toks)
        lane.rollback_to(f0)
    cap = 1 << 18
    buf = torch.zeros(5 * cap * 3, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    assert lib.hs_cta_trace(buf.data_ptr(), cap) == 0, "needs a trace build"
    lane._forward(toks)
    torch.cuda.synchronize()
    lib.hs_cta_trace(None, 0)
    lane.rollback_to(f0)
    rec = buf[4 * cap * 3:].view(-1, 16).cpu().numpy().astype(np.uint64)
    rec = rec[rec[:, 15] > 0]
    if a.raw:
        np.save(a.raw, rec)
    ident = rec[:, 0]
    ntiles = (ident >> np.uint64(48)).astype(int)
    split = ((ident >> np.uint64(16)) & np.uint64(0xffff)).astype(int)
    # columns: start, release, first, last, accum, (final), tmem, yres, csync1, dsmem, finalize, end
    r = rec.astype(np.int64)
    ts = np.stack([r[:, 1], r[:, 2], r[:, 3], r[:, 4], r[:, 5], r[:, 6], r[:, 7], r[:, 8], r[:, 9], r[:, 10],
                   r[:, 12], r[:, 13], r[:, 14], r[:, 11], r[:, 15]], axis=1)
    # group into launches: consecutive (by release time) CTAs of the same tile count
    order = np.argsort(ts[:, 1], kind="stable")
    groups, cur = [], None
    for i in order:
        if cur is None or ntiles[i] != cur[0] or ts[i, 1] > cur[2] + 3000:
            cur = [ntiles[i], [], ts[i, 1]]
            groups.append(cur)
        cur[1].append(i)
        cur[2] = max(cur[2], ts[i, 1])
    names = ["start", "release", "first", "last", "accum", "final", "tmem", "yres", "csync1", "dsmem", "stores",
             "wsum", "bar", "fin", "end"]
    kinds = collections.defaultdict(list)
    prev_end = None
    for nt, idx, _ in groups:
        idx = np.array(idx)
        r0 = ts[idx, 1].min()
        ks = split[idx].max() + 1
        row = {}
        row["start_med"] = np.median(ts[idx, 0] - r0) / 1e3
        for j, n in enumerate(names[1:], start=1):
            col = ts[idx, j]
            col = col[col > 0]
            v = (col - r0) / 1e3 if len(col) else np.array([np.nan])
            row[n + "_p50"] = np.median(v)
            row[n + "_max"] = v.max()
        row["gap_prev_end_to_release"] = (r0 - prev_end) / 1e3 if prev_end is not None else float("nan")
        prev_end = ts[idx, 14].max()
        kinds[(nt, ks, len(idx))].append(row)
    print(f"lane {a.lane} t={a.t}: {len(groups)} GEMV launches; times in us relative to the launch's first release "
          "(medians over launches of the per-launch p50 / max over CTAs)")
    print(f"{'tiles x ks (ctas)':>20s} {'n':>3s} {'start':>7s} " + " ".join(f"{n:>7s}" for n in names[1:])
          + f" {'endmax':>7s} {'gap':>6s}")
    for (nt, ks, nc), rows in sorted(kinds.items(), key=lambda x: -x[0][0] * x[0][1]):
        med = {k: np.nanmedian([r[k] for r in rows]) for k in rows[0]}
        print(f"{f'{nt} x {ks} ({nc})':>20s} {len(rows):3d} {med['start_med']:7.2f} "
              + " ".join(f"{med[n + '_p50']:7.2f}" for n in names[1:])
              + f" {med['end_max']:7.2f} {med['gap_prev_end_to_release']:6.2f}")


if __name__ == "__main__":
    main()
