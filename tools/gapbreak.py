#!/usr/bin/env python3
"""Host-time breakdown of the gap between a round's read-back and its next
native launch (the GPU idles for that long): wall-clock marks at the end of
_readback, at entry of the session-level helpers and at the first call of
each C entry point after it, averaged over a generate() at the Llama2-7B
shape (32K context by default).

    python tools/gapbreak.py [--ctx 32768] [--gen 96]
"""
from __future__ import annotations

import argparse
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--gen", type=int, default=96)
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200 import _abi, model as M, speculation as S

    tdm = P.DeviceModel.random(P.ModelConfig(**{**bench.TARGET_7B, "max_seq": a.ctx + 4096}), seed=1)
    ddm = P.DeviceModel.random(P.ModelConfig(**{**bench.DRAFT_68M, "max_seq": a.ctx + 4096}), seed=1001)
    tdm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    ddm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    tw, dw = P.ModelWeights.on_device(tdm), P.ModelWeights.on_device(ddm)
    ctx = np.random.default_rng(0).integers(1, 32000, a.ctx).tolist()
    spec = P.SpecConfig(target_len=a.ctx + 1, gamma1=2, gamma2=4, streaming=P.StreamingConfig(n_sink=4, budget=256),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
    sess.config.target_len = len(sess.committed) + 32
    sess.generate(seed=1)

    marks = collections.defaultdict(list)   # label -> [us after the read-back]
    state = {"t0": None, "seen": set()}

    def mark(label):
        if state["t0"] is not None and label not in state["seen"]:
            state["seen"].add(label)
            marks[label].append((time.perf_counter() - state["t0"]) * 1e6)

    def wrap_py(mod, name):
        f = getattr(mod, name)

        def w(*args, **kw):
            mark("py:" + name)
            return f(*args, **kw)
        setattr(mod, name, w)

    orig_rb = S._readback

    def rb(*args, **kw):
        out = orig_rb(*args, **kw)
        state["t0"] = time.perf_counter()
        state["seen"] = set()
        return out
    S._readback = rb
    for n in ("_inner_round_dev", "_draft_round_dev", "_score_rows_dev", "_chain_dev"):
        wrap_py(S, n)
    wrap_py(M, "forward_device")
    S.forward_device = M.forward_device
    lib = _abi.lib

    class Spy:
        def __init__(self, inner):
            self._inner = inner

        def __getattr__(self, name):
            f = getattr(self._inner, name)
            if not name.startswith("hs_") or not callable(f):
                return f

            def w(*args):
                mark("c:" + name)
                mark("c:(first native call)")
                return f(*args)
            return w
    spy = Spy(lib)
    for mod in (S, M, P.caches):
        if hasattr(mod, "lib"):
            mod.lib = spy
    orig_replay = torch.cuda.CUDAGraph.replay

    def replay(self):
        mark("graph.replay")
        mark("c:(first native call)")
        return orig_replay(self)
    torch.cuda.CUDAGraph.replay = replay

    sess.config.target_len = len(sess.committed) + a.gen
    sess.generate(seed=2)
    torch.cuda.synchronize()
    rows = sorted(((float(np.median(v)), k, len(v)) for k, v in marks.items()))
    print(f"{'median us':>10} {'n':>4}  first occurrence after a read-back")
    for med, k, n in rows:
        print(f"{med:10.1f} {n:4d}  {k}")


if __name__ == "__main__":
    main()
