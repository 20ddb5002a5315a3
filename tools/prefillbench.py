#!/usr/bin/env python3
"""Prefill throughput at the Llama2-7B shape: hs_prefill (GEMM prefill) vs the
row-exact decode path, device time with CUDA events.

    python tools/prefillbench.py [--t 4096 16384]
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
    ap.add_argument("--t", type=int, nargs="+", default=[2048, 8192, 16384])
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200 import model as M
    tw = P.ModelWeights.on_device(P.DeviceModel.random(P.ModelConfig(**{**bench.TARGET_7B, "max_seq": max(a.t) + 64}), 1))
    out = {}
    for t in a.t:
        toks = np.random.default_rng(t).integers(1, 32000, t).tolist()
        res = {}
        for name, pre in (("gemm_prefill", True), ("decode_path", False)):
            if not pre and t > 4096:
                continue
            cache = P.FullCache.from_config(tw.config)
            logits = torch.empty((t, 32000), device="cuda")
            M.forward_device(tw, toks[:128], cache, out=logits[:128], prefill=pre)   # warm
            cache.rollback_to(0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            M.forward_device(tw, toks, cache, out=logits, prefill=pre)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            res[name] = {"ms": ms, "tokens_per_s": t / ms * 1e3}
            del cache
            torch.cuda.empty_cache()
        out[f"t{t}"] = res
        print(json.dumps({f"t{t}": res}), flush=True)


if __name__ == "__main__":
    main()
