#!/usr/bin/env python3
"""GPU idle time of a decode step without a profiler in the loop (trace build:
HS_TRACE_BUILD=1 python paper_2404_11912_b200/build.py --force).  Every CTA of
the library's kernels records its start / end (globaltimer); the union of
those intervals is the time the GPU had work of ours resident, the rest of
the generate() span is idle (host gaps, syncs, launch latency).  The union
over-counts busy time (a CTA waiting on griddepcontrol counts), so the idle
figure is a lower bound... of idle; copies issued by torch are not kernels
of ours and count as idle.

    python tools/idle_trace.py [--ctx 122880] [--gen 32]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=122880)
    ap.add_argument("--gen", type=int, default=32)
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200._abi import lib
    lib.hs_cta_trace.restype = C.c_int
    lib.hs_cta_trace.argtypes = [C.c_void_p, C.c_uint]
    tdm = P.DeviceModel.random(P.ModelConfig(**bench.TARGET_7B), seed=1)
    ddm = P.DeviceModel.random(P.ModelConfig(**bench.DRAFT_68M), seed=1001)
    tdm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    ddm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    tw, dw = P.ModelWeights.on_device(tdm), P.ModelWeights.on_device(ddm)
    ctx = np.random.default_rng(0).integers(1, 32000, a.ctx).tolist()
    spec = P.SpecConfig(target_len=a.ctx + 1, gamma1=2, gamma2=4, streaming=P.StreamingConfig(n_sink=4, budget=256),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
    sess.config.target_len = len(sess.committed) + 32
    sess.generate(seed=1)                      # warm-up: graphs captured, workspaces grown
    cap = 1 << 21
    buf = torch.zeros(5 * cap * 3, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    assert lib.hs_cta_trace(buf.data_ptr(), cap) == 0, "needs a trace build"
    sess.config.target_len = len(sess.committed) + a.gen
    t0 = time.perf_counter()
    sess.generate(seed=2)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e6
    lib.hs_cta_trace(None, 0)
    rec = buf[:4 * cap * 3].view(-1, 3).cpu().numpy().astype(np.uint64)
    rec = rec[rec[:, 1] > 0]
    s = rec[:, 1].astype(np.int64)
    e = rec[:, 2].astype(np.int64)
    order = np.argsort(s)
    s, e = s[order], e[order]
    busy, cur_s, cur_e = 0, s[0], e[0]
    gaps = []
    for a_, b_ in zip(s[1:], e[1:]):
        if a_ > cur_e:
            busy += cur_e - cur_s
            gaps.append(a_ - cur_e)
            cur_s, cur_e = a_, b_
        else:
            cur_e = max(cur_e, b_)
    busy += cur_e - cur_s
    span = e.max() - s.min()
    gaps = np.array(gaps) / 1e3
    print(f"generate({a.gen} tokens) at {a.ctx}: {len(rec)} CTA records, span {span / 1e3:.1f} us "
          f"(host wall {wall:.0f} us), busy {busy / 1e3:.1f} us, idle {(span - busy) / 1e3:.1f} us "
          f"= {100 * (span - busy) / span:.2f}%")
    big = gaps[gaps > 5]
    print(f"idle gaps > 5 us: {len(big)}, total {big.sum():.1f} us, median {np.median(big) if len(big) else 0:.1f} us; "
          f"gaps <= 5 us: {len(gaps) - len(big)}, total {gaps[gaps <= 5].sum():.1f} us")


if __name__ == "__main__":
    main()
