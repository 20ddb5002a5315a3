#!/usr/bin/env python3
"""chunk_score device time at the Llama2-7B shape (32 layers x 32 kv heads x
122,880 keys, chunk 8; CUDA events, no profiler) for the TMA-staged kernel and
the generic one (HS_SCORE_NO_TMA=1 in a second process), plus an equality
check of the two paths' scores (fp64, must agree to 1e-12 relative).

    python tools/scorebench.py [--layers 32] [--ctx 122880] [--chunk 8] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(a):
    import torch
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200._abi import check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr
    L, n = a.layers, a.ctx
    full = P.FullCache(L, 32, 128, n + 64)
    full.fill_random_(n, seed=0)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    q = torch.randn((L, 32, 128), device="cuda", generator=g)
    nch = (n + a.chunk - 1) // a.chunk
    out = torch.empty((L, nch), dtype=torch.float64, device="cuda")

    def call():
        check(lib.hs_chunk_score(ptr(full.k), 1, 32 * full.cap * 128, full.cap * 128, 128, L, 32, 128, n, a.chunk,
                                 ptr(q), 32, ptr(out), stream_ptr()))
    call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    nbytes = L * 32 * n * 128 * 2
    torch.save(out.cpu(), a.save)
    return {"ms": ms, "GBps": nbytes / ms / 1e6, "bytes": nbytes}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=122880)
    ap.add_argument("--chunk", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--save", default="/tmp/scores.pt")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(run(a)))
        return
    import torch
    res = {}
    for name, env in (("tma", {}), ("generic", {"HS_SCORE_NO_TMA": "1"})):
        save = f"/tmp/scores_{name}.pt"
        cmd = [sys.executable, __file__, "--child", "--layers", str(a.layers), "--ctx", str(a.ctx), "--chunk",
               str(a.chunk), "--reps", str(a.reps), "--save", save]
        r = subprocess.run(cmd, env={**os.environ, **env}, capture_output=True, text=True)
        if r.returncode:
            print(r.stderr[-3000:])
            raise SystemExit(f"{name} failed")
        res[name] = json.loads(r.stdout.strip().splitlines()[-1])
    x, y = torch.load("/tmp/scores_tma.pt"), torch.load("/tmp/scores_generic.pt")
    rel = ((x - y).abs().max() / y.abs().max()).item()
    same_rank = bool((torch.argsort(-x, dim=1, stable=True)[:, :512] == torch.argsort(-y, dim=1, stable=True)[:, :512]).all())
    res["max_rel_diff"] = rel
    res["top512_identical"] = same_rank
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
