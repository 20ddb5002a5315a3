#!/usr/bin/env python3
"""Device time of single lane forwards at the Llama2-7B shape (CUDA events,
no profiler): retrieval lane t=3, full lane t=7 (context --ctx), draft t=1, and
the draft's captured step graph replayed back to back (draft_graph).

    python tools/fwdbench.py [--ctx 16384] [--reps 10]
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
    ap.add_argument("--ctx", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import paper_2404_11912_b200 as P
    import bench
    tdm = P.DeviceModel.random(P.ModelConfig(**bench.TARGET_7B), seed=1)
    tw = P.ModelWeights.on_device(tdm)
    dw = P.ModelWeights.on_device(P.DeviceModel.random(P.ModelConfig(**bench.DRAFT_68M), seed=2))
    ctx = np.random.default_rng(0).integers(1, 32000, a.ctx).tolist()
    spec = P.SpecConfig(target_len=a.ctx + 64, gamma1=2, gamma2=4,
                        streaming=P.StreamingConfig(n_sink=4, budget=256),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
    out = {}
    for name, lane, t in (("retr_t3", sess.retr_lane, 3), ("retr_t1", sess.retr_lane, 1), ("full_t7", sess.full_lane, 7),
                          ("draft_t1", sess.draft_lane, 1)):
        toks = torch.ones(t, dtype=torch.int32, device="cuda")
        f0 = lane.frontier
        for _ in range(3):
            lane._forward(toks)
            lane.rollback_to(f0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            lane._forward(toks)
            lane.rollback_to(f0)
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / a.reps
    # the draft lane's captured one-token step, replayed back to back (device
    # time of the step as the decode loop runs it: no host launches inside)
    sg = sess.draft_lane.step_graph()
    for _ in range(3):
        sg.graph.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps * 5):
        sg.graph.replay()
    e1.record()
    torch.cuda.synchronize()
    out["draft_graph"] = e0.elapsed_time(e1) / (a.reps * 5)
    w = tw.device().weight_bytes
    out["dense_GBps_retr_t3"] = w / (out["retr_t3"] * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
