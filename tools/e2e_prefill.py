#!/usr/bin/env python3
"""End to end with a real prompt instead of bench.py's synthetic caches:
HierarchicalSession(target, draft, prompt) prefills the full cache (GEMM
prefill + tensor-core prefill attention), the draft's StreamingLLM cache and
builds the retrieval cache, then generate() decodes --gen tokens.  Planted-
successor weights as in bench.py (random prompt tokens).

    python tools/e2e_prefill.py [--context 122880] [--gen 128]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=122880)
    ap.add_argument("--gen", type=int, default=128)
    a = ap.parse_args()
    import bench
    import paper_2404_11912_b200 as P
    seq = a.context + a.gen + 64
    tdm = P.DeviceModel.random(P.ModelConfig(**{**bench.TARGET_7B, "max_seq": seq}), 1)
    ddm = P.DeviceModel.random(P.ModelConfig(**{**bench.DRAFT_68M, "max_seq": seq}), 1001)
    tdm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    ddm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    tw, dw = P.ModelWeights.on_device(tdm), P.ModelWeights.on_device(ddm)
    prompt = np.random.default_rng(0).integers(1, 32000, a.context).tolist()
    spec = P.SpecConfig(target_len=a.context + a.gen, gamma1=bench.GAMMA1, gamma2=bench.GAMMA2,
                        streaming=P.StreamingConfig(n_sink=bench.SINK, budget=bench.STREAM),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess = P.HierarchicalSession(tw, dw, prompt, spec)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    out, trace = sess.generate()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s = trace.summary()
    res = {"context": a.context, "prefill_and_build_s": t1 - t0, "gen_tokens": len(out) - a.context,
           "decode_ms_per_token": (t2 - t1) * 1e3 / (len(out) - a.context),
           "inner_rate": s["inner"]["accepted"] / max(1, s["inner"]["proposed"]),
           "outer_rate": s["outer"]["accepted"] / max(1, s["outer"]["proposed"])}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
