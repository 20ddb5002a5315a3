#!/usr/bin/env python3
"""Minimal workloads for `ncu --set full` captures of single kernels at the
Llama2-7B shape (4 layers; every launch of a kernel name in one run is the
same shape, so --launch-skip picks a warm one):

    python tools/ncu_targets.py retrieval   # retrieval-view forward, t = 3:
                                            #   per layer gemv wqkv, attn_tc (288 items) + combine,
                                            #   gemv w_o, gemv gate|up, gemv w_down
    python tools/ncu_targets.py score       # chunk_score over 122,880 keys (2 layers)
    python tools/ncu_targets.py full        # verify forward, t = 7, over a 122,880-key full cache
                                            #   (attn_tc 60 splits + combine<64>)

GEMV launch order per layer: wqkv, w_o, gate|up, w_down (lm_head once per
forward), so with L layers and F warm forwards skip F*(4L+1) + k to land on
matrix k of layer 0.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "retrieval"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    import paper_2404_11912_b200 as P
    L = 4
    cfg = P.ModelConfig(n_layers=L, n_heads=32, n_kv_heads=32, head_dim=128, d_ff=11008, vocab_size=32000,
                        max_seq=131072)
    if what == "retrieval":
        tw = P.ModelWeights.on_device(P.DeviceModel.random(cfg, seed=1))
        n = 16384
        full = P.FullCache.from_config(cfg)
        full.fill_random_(n, seed=0)
        rc = P.RetrievalCache.from_config(cfg, P.RetrievalConfig(chunk_size=8, budget=4096))
        q = torch.randn((L, 32, 128), device="cuda")
        rc.build(full, q, n)
        lane = P.speculation.Lane(tw, rc)
        toks = torch.ones(3, dtype=torch.int32, device="cuda")
        f0 = rc.frontier
        for _ in range(reps):
            lane._forward(toks)
            lane.rollback_to(f0)
        torch.cuda.synchronize()
    elif what == "full":
        tw = P.ModelWeights.on_device(P.DeviceModel.random(cfg, seed=1))
        n = 122880
        full = P.FullCache.from_config(cfg)
        full.fill_random_(n, seed=0)
        lane = P.speculation.Lane(tw, full)
        toks = torch.ones(7, dtype=torch.int32, device="cuda")
        f0 = full.frontier
        for _ in range(reps):
            lane._forward(toks)
            lane.rollback_to(f0)
        torch.cuda.synchronize()
    elif what == "score":
        from paper_2404_11912_b200._abi import check, lib
        from paper_2404_11912_b200.runtime import ptr, stream_ptr
        n = 122880
        full = P.FullCache(2, 32, 128, n + 64)
        full.fill_random_(n, seed=0)
        q = torch.randn((2, 32, 128), device="cuda")
        nch = n // 8
        out = torch.empty((2, nch), dtype=torch.float64, device="cuda")
        for _ in range(reps):
            check(lib.hs_chunk_score(ptr(full.k), 1, 32 * full.cap * 128, full.cap * 128, 128, 2, 32, 128, n, 8,
                                     ptr(q), 32, ptr(out), stream_ptr()))
        torch.cuda.synchronize()
    else:
        raise SystemExit(f"unknown target {what}")


if __name__ == "__main__":
    main()
