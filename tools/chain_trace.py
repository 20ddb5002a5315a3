#!/usr/bin/env python3
"""Event trace of the persistent dense-chain kernel (debug aid): runs one
retrieval-lane forward at the Llama2-7B shape and prints, per phase of the
last chain launch, when CTAs issue weights, start MMAs, finish builds and
epilogues and pass the grid barriers (us from the earliest event)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def per_cta(tr, t0, phase):
    """per-CTA epilogue completion times of one phase (us)"""
    import numpy as np
    out = []
    for c in range(tr.shape[0]):
        ev = tr[c]
        sel = (ev[:, 0] == 500 + phase) & (ev[:, 1] >= t0)
        ts = np.sort((ev[sel, 1] - t0) / 1e3)
        out.append((c, ts))
    return out


def main():
    import paper_2404_11912_b200 as P
    import bench
    from paper_2404_11912_b200._abi import lib
    lib.hs_chain_trace.restype = C.c_int
    lib.hs_chain_trace.argtypes = [C.c_void_p]
    tw = P.ModelWeights.on_device(P.DeviceModel.random(P.ModelConfig(**{**bench.TARGET_7B, "n_layers": 2}), seed=1))
    cache = P.FullCache.from_config(tw.config)
    cache.fill_random_(4096)
    t = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    toks = torch.ones(t, dtype=torch.int32, device="cuda")
    for _ in range(2):
        P.model.forward_device(tw, toks, cache)
        cache.rollback_to(4096)
    buf = torch.zeros(148 * 128 * 2, dtype=torch.int64, device="cuda")
    lib.hs_chain_trace(buf.data_ptr())
    P.model.forward_device(tw, toks, cache)
    torch.cuda.synchronize()
    lib.hs_chain_trace(None)
    tr = buf.view(148, 128, 2).cpu().numpy()
    ev = tr[tr[:, :, 1] > 0]
    starts = ev[ev[:, 0] == 1][:, 1]
    t0 = starts.min()                       # the last chain launch (slots are reused per launch)
    ev = ev[ev[:, 1] >= t0]
    names = {1: "producer start", 100: "W first issue", 200: "MMA phase start", 300: "B built", 400: "barrier passed",
             500: "epilogue done", 600: "phase arrive"}
    rows = {}
    for code, ns in ev:
        base = code if code < 100 else code - code % 100
        ph = 0 if code < 100 else code % 100
        rows.setdefault((base, ph), []).append((ns - t0) / 1e3)
    for ph in (1, 3):
        cts = per_cta(tr, t0, ph)
        cts.sort(key=lambda x: -(x[1].max() if len(x[1]) else 0))
        print(f"phase {ph} slowest CTAs (cta: item completion us):")
        for c, ts in cts[:6] + cts[-3:]:
            print(f"   cta {c:3d}: " + " ".join(f"{x:6.1f}" for x in ts))
        n = np.array([len(ts) for _, ts in cts])
        print(f"   items per CTA: min {n.min()} max {n.max()} mean {n.mean():.2f}")
    for (base, ph), v in sorted(rows.items(), key=lambda x: (x[0][1], min(x[1]))):
        v = np.array(v)
        print(f"phase {ph} {names.get(base, base):16s} n={len(v):4d}  first {v.min():8.2f}  median {np.median(v):8.2f}  "
              f"last {v.max():8.2f} us")


if __name__ == "__main__":
    main()
