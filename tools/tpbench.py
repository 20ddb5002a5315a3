#!/usr/bin/env python3
"""Per-rank dense-path time of a tensor-parallel forward at the Llama2-7B
shape (hs_forward_tp's row blocks), measured on one GPU: rank 0's block of
every projection (wqkv, w_o, gate|up, w_down per layer, lm_head) as the same
GEMV launches the forward issues, back to back with CUDA events, for G = 1, 2,
4, 8.  The exchanges (all-gathers over NVLink) are not measurable here; the
output states the weight-streaming part only.

    python tools/tpbench.py [--t 3] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def rows(N, rank, world):
    tiles = (N + 127) // 128
    t0, t1 = tiles * rank // world, tiles * (rank + 1) // world
    return t0 * 128, max(0, min(N, t1 * 128) - t0 * 128)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, default=3)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200._abi import check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr
    cfg = P.ModelConfig(**bench.TARGET_7B)
    dm = P.DeviceModel.random(cfg, seed=1)
    d, ff, V = cfg.d_model, cfg.d_ff, cfg.vocab_size
    s = stream_ptr()
    xs = torch.zeros((24, dm.ld_ff), dtype=torch.bfloat16, device="cuda")
    xo = torch.zeros((24, dm.ld_ff), dtype=torch.bfloat16, device="cuda")
    y = torch.zeros((8, V), device="cuda")
    out = {}
    for G in (1, 2, 4, 8):
        calls = []
        mats = [("wqkv", dm.wqkv, 12288, dm.ld_d, 0), ("wo", dm.wo, d, dm.ld_d, 1), ("wgu", dm.wgu, 2 * ff, dm.ld_d, 2),
                ("wdown", dm.wdown, d, dm.ld_ff, 1)]
        wbytes = 0
        for layer in range(cfg.n_layers):
            for name, w, N, ld, epi in mats:
                r0, n = rows(N, 0, G)
                calls.append((w[layer], r0, n, ld, epi))
                wbytes += n * (d if ld == dm.ld_d else ff) * 2
        r0, n = rows(V, 0, G)
        calls.append((dm.head, r0, n, dm.ld_d, 0))
        wbytes += n * d * 2
        ws = {}
        for (w, r0, n, ld, epi) in calls:
            nb = lib.hs_gemv_tc_workspace_bytes(n, ld)
            if nb not in ws:
                ws[nb] = torch.zeros(nb, dtype=torch.uint8, device="cuda")

        def run():
            for (w, r0, n, ld, epi) in calls:
                nb = lib.hs_gemv_tc_workspace_bytes(n, ld)
                check(lib.hs_gemv_tc(ptr(xs), a.t, ptr(w) + r0 * ld * 2, ld, n, epi, ptr(y) if epi != 2 else None,
                                     n, ptr(xo) if epi == 2 else None, dm.ld_ff, ptr(ws[nb]), nb, s))
        run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        out[f"G{G}"] = {"rank0_dense_ms": ms, "weight_GB": wbytes / 1e9, "GBps": wbytes / ms / 1e6,
                        "launches": len(calls)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
