#!/usr/bin/env python3
"""Debug aid: randomized-forward case 2 (dh 128, H 1, 2 layers) GEMM prefill vs the oracle; run with and
without HS_NO_PDL=1 to separate a dependency race from arithmetic."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def main():
    import paper_2404_11912_b200 as P
    from oracle import hs_oracle as O
    from tests.test_gpu_session import bf16_weights
    for L, dff, plen in ((2, 96, 314), (2, 96, 64), (2, 96, 130), (2, 352, 314), (3, 96, 314)):
        cfg = P.ModelConfig(n_layers=L, n_heads=1, n_kv_heads=1, head_dim=128, d_ff=dff, vocab_size=300, max_seq=1024)
        w = bf16_weights(P, P.generate_weights(cfg, 502, tied_head=False))
        om = O.OModel(O.OConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__}), O.round_weights_bf16(w.tensors), False)
        prompt = np.random.default_rng(1).integers(1, 300, plen).tolist()
        errs = []
        for rep in range(3):
            g = P.prefill(w, prompt, P.FullCache.from_config(cfg))
            r = O.prefill(om, prompt, O.OFullCache(L, 1, 128, 1024, kv_bf16=True))
            d = np.abs(g - r)
            errs.append((d.max() / np.abs(r).max(), int(np.argmax(d.max(-1)))))
        print(f"L{L} dff{dff} plen{plen} NO_PDL={os.environ.get('HS_NO_PDL', '0')}: rel err, worst row per rep {errs}",
              flush=True)


if __name__ == "__main__":
    main()
