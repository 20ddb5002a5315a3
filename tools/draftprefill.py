#!/usr/bin/env python3
"""Device time of the draft lane's prefill (JF68M shape, StreamingLLM cache)
over a long prompt: the reference processes it token by token
(caches.py:230); here it goes through the row-exact decode path in 8-row
blocks with the per-query sink + window exposure.

    python tools/draftprefill.py [--t 16384 122880]
"""
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
    ap.add_argument("--t", type=int, nargs="+", default=[16384])
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    dw = P.ModelWeights.on_device(P.DeviceModel.random(P.ModelConfig(**{**bench.DRAFT_68M,
                                                                       "max_seq": max(a.t) + 64}), 2))
    for t in a.t:
        toks = np.random.default_rng(t).integers(1, 32000, t).tolist()
        lane = P.Lane(dw, P.StreamingCache.from_config(dw.config, P.StreamingConfig(n_sink=4, budget=256)))
        lane.prefill(toks[:64])
        lane = P.Lane(dw, P.StreamingCache.from_config(dw.config, P.StreamingConfig(n_sink=4, budget=256)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        lane.prefill(toks)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({f"t{t}": {"ms": ms, "tokens_per_s": t / ms * 1e3}}), flush=True)


if __name__ == "__main__":
    main()
