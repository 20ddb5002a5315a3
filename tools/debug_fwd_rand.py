#!/usr/bin/env python3
"""Debug aid: the randomized-forward test's cases, printing where the GPU
prefill / decode rows deviate most from the oracle (GEMM prefill vs the
row-exact decode path for the prompt)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def main():
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200 import model as M
    from oracle import hs_oracle as O
    from tests.test_gpu_session import bf16_weights
    rng = np.random.default_rng(77)
    for case in range(6):
        dh = int(rng.choice([64, 128]))
        kvh = int(rng.choice([1, 2, 4]))
        H = kvh * int(rng.choice([1, 2, 4]))
        cfg = P.ModelConfig(n_layers=2, n_heads=H, n_kv_heads=kvh, head_dim=dh, d_ff=int(rng.integers(3, 12)) * 32,
                            vocab_size=300, max_seq=1024)
        w = bf16_weights(P, P.generate_weights(cfg, 500 + case, tied_head=bool(case % 2)))
        om = O.OModel(O.OConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__}),
                      O.round_weights_bf16(w.tensors), w.tied_head)
        plen = int(rng.integers(20, 400))
        prompt = rng.integers(1, 300, plen).tolist()
        rng.integers(1, 300, int(rng.integers(2, 12)))
        rng.integers(1, 300, 3)
        want = O.prefill(om, prompt, O.OFullCache(2, kvh, dh, 1024, kv_bf16=True))
        for mode in ("gemm", "rowexact"):
            keep = M.PREFILL_MIN_ROWS
            if mode == "rowexact":
                M.PREFILL_MIN_ROWS = 10 ** 9
            try:
                g = P.prefill(w, prompt, P.FullCache.from_config(cfg))
            finally:
                M.PREFILL_MIN_ROWS = keep
            d = np.abs(g - want)
            i = np.unravel_index(np.argmax(d), d.shape)
            print(f"case {case} dh {dh} H {H} kvh {kvh} dff {cfg.d_ff} plen {plen} {mode}: max err {d.max():.3g} "
                  f"at {i} (got {g[i]:.6g} want {want[i]:.6g}); rel {d.max() / np.abs(want).max():.3g}; "
                  f"rows with err > 1e-3: {int((d.max(-1) > 1e-3).sum())}", flush=True)


if __name__ == "__main__":
    main()
