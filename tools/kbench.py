#!/usr/bin/env python3
"""Kernel micro-benchmark at the Llama2-7B shapes (CUDA events on the
launching stream, inputs larger than L2 or rotated across layers).

    python tools/kbench.py [--layers 4] [--ctx 122880] [--json out.json]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for r in range(reps):
        fn(r)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--ctx", type=int, default=122880)
    ap.add_argument("--json", default=None)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200._abi import HsStep, check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr, workspaces

    L = a.layers
    cfg = P.ModelConfig(n_layers=L, n_heads=32, n_kv_heads=32, head_dim=128, d_ff=11008, vocab_size=32000,
                        max_seq=131072)
    dm = P.DeviceModel.random(cfg, seed=1)
    d, ff = 4096, 11008
    out = {"gemv": {}, "attn": {}}
    s = stream_ptr()
    shapes = {"wqkv": (dm.wqkv, 12288, d, dm.ld_d, 0), "wo": (dm.wo, d, d, dm.ld_d, 1),
              "wgu": (dm.wgu, 2 * ff, d, dm.ld_d, 2), "wdown": (dm.wdown, d, ff, dm.ld_ff, 1),
              "head": (dm.head.unsqueeze(0), 32000, d, dm.ld_d, 0)}
    xs = torch.zeros((24, dm.ld_ff), dtype=torch.bfloat16, device="cuda")
    xo = torch.zeros((24, dm.ld_ff), dtype=torch.bfloat16, device="cuda")
    y = torch.zeros((8, 32000), device="cuda")
    for t in (1, 3, 5, 8):
        for name, (w, N, K, ld, epi) in shapes.items():
            if a.only and a.only not in name:
                continue
            nb = lib.hs_gemv_tc_workspace_bytes(N, ld)
            ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
            nl = w.shape[0]

            def fn(r, w=w, N=N, ld=ld, epi=epi, nb=nb, ws=ws, nl=nl):
                check(lib.hs_gemv_tc(ptr(xs), t, ptr(w[r % nl]), ld, N, epi, ptr(y) if epi != 2 else None,
                                     N, ptr(xo) if epi == 2 else None, dm.ld_ff, ptr(ws), nb, s))
            us = timeit(fn)
            out["gemv"][f"{name}_t{t}"] = {"us": us, "GBps": N * K * 2 / us / 1e3}
    # attention over a full cache
    if not a.only or "attn" in a.only:
        n = a.ctx
        cache = P.FullCache(2, 32, 128, n + 64)
        for l in range(2):
            cache.k[l, :, :n].normal_()
            cache.v[l, :, :n].normal_()
        for t in (1, 3, 5, 8):
            q = torch.randn((t, 32, 128), device="cuda")
            o = torch.empty((t, 4096), device="cuda")
            st = HsStep()
            st.pos0, st.n_view, st.split = n - t, n, P.caches.FULL_SPLIT
            nb = lib.hs_attention_workspace_bytes(t, 32, 128, n, st.split)
            ws = workspaces.get("kb", nb)

            def fa(r):
                check(lib.hs_attention(cache._ref, r % 2, C.byref(st), 32, ptr(q), t, ptr(o), ptr(ws), nb, s))
            us = timeit(fa, reps=10)
            out["attn"][f"full_t{t}"] = {"us": us, "GBps": n * 32 * 128 * 4 / us / 1e3}
        # retrieval-sized view (4,096 + tail)
        rn = 4100
        st2 = HsStep()
        for t in (1, 3):
            st2.pos0, st2.n_view, st2.split = n - t, rn, P.caches.SMALL_SPLIT
            q = torch.randn((t, 32, 128), device="cuda")
            o = torch.empty((t, 4096), device="cuda")
            nb = lib.hs_attention_workspace_bytes(t, 32, 128, rn, st2.split)
            ws = workspaces.get("kb2", nb)

            def fr(r):
                check(lib.hs_attention(cache._ref, r % 2, C.byref(st2), 32, ptr(q), t, ptr(o), ptr(ws), nb, s))
            us = timeit(fr)
            out["attn"][f"retr_t{t}"] = {"us": us, "GBps": rn * 32 * 128 * 4 / us / 1e3}
    print(json.dumps(out, indent=1))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
