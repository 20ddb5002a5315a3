#!/usr/bin/env python3
"""Host time between each round's device->host sync and the next kernel
launch (the GPU idles for that long), at the Llama2-7B shape."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import bench
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200 import model as M
    from paper_2404_11912_b200 import speculation as S
    tdm, ddm = P.DeviceModel.random(P.ModelConfig(**bench.TARGET_7B), 1), P.DeviceModel.random(
        P.ModelConfig(**bench.DRAFT_68M), 1001)
    tdm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    ddm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
    tw, dw = P.ModelWeights.on_device(tdm), P.ModelWeights.on_device(ddm)
    ctx = np.random.default_rng(0).integers(1, 32000, 16384).tolist()
    spec = P.SpecConfig(target_len=16385, gamma1=2, gamma2=4, streaming=P.StreamingConfig(n_sink=4, budget=256),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
    sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
    gaps, last = [], [None]
    real_rb, real_fd, real_ds = S._readback, M.forward_device, S.lib.hs_draft_sample

    def rb(*a, **k):
        out = real_rb(*a, **k)
        last[0] = time.perf_counter()
        return out

    def first_launch():
        if last[0] is not None:
            gaps.append(time.perf_counter() - last[0])
            last[0] = None

    def fd(*a, **k):
        first_launch()
        return real_fd(*a, **k)

    class DS:
        def __call__(self, *a):
            first_launch()
            return real_ds(*a)

    S._readback, S.forward_device = rb, fd
    S.lib.hs_draft_sample = DS()
    for i in range(4):
        sess.config.target_len = len(sess.committed) + 32
        t0 = time.perf_counter()
        sess.generate(seed=i)
        torch.cuda.synchronize()
    S._readback, S.forward_device = real_rb, real_fd
    g = np.array(gaps[len(gaps) // 4:]) * 1e6
    print(f"syncs {len(g)}: host gap after sync median {np.median(g):.1f} us, mean {g.mean():.1f} us, "
          f"p90 {np.percentile(g, 90):.1f} us")


if __name__ == "__main__":
    main()
