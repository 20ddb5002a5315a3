#!/usr/bin/env python3
"""Debug aid for the prefill GEMM: (1) hs_gemm3_tc alone at prefill-like
shapes with plane stride == K; (2) a 1-layer prefill's cached K/V against the
oracle's (bf16 values: count mismatches beyond rounding flips)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200._abi import check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr
    from oracle import hs_oracle as O
    from tests.test_gpu_kernels import _split3_host, _bf16
    rng = np.random.default_rng(0)
    for R, K, N in ((314, 128, 384), (314, 128, 300), (314, 128, 192), (80, 512, 1536), (2048, 4096, 4096)):
        x = rng.normal(0, 1, (R, K)).astype(np.float32)
        W = _bf16(rng.normal(0, 0.02, (N, K)).astype(np.float32))
        planes = [torch.from_numpy(p).cuda().to(torch.bfloat16).contiguous() for p in _split3_host(x)]
        Wd = torch.from_numpy(W).cuda().to(torch.bfloat16).contiguous()
        y = torch.zeros((R, N), device="cuda")
        check(lib.hs_gemm3_tc(ptr(planes[0]), ptr(planes[1]), ptr(planes[2]), K, R, ptr(Wd), K, N, ptr(y), N, 0,
                              stream_ptr()))
        ref = x.astype(np.float64) @ W.astype(np.float64).T
        d = np.abs(y.cpu().numpy() - ref)
        h = np.abs(planes[0].float().cpu().numpy().astype(np.float64) @ W.astype(np.float64).T - ref)
        print(f"gemm R{R} K{K} N{N}: max rel err {d.max() / np.abs(ref).max():.3g} (hi plane only would be "
              f"{h.max() / np.abs(ref).max():.3g}); worst row {np.unravel_index(np.argmax(d), d.shape)}", flush=True)
    for dh, H, kvh, dff in ((128, 1, 1, 96), (64, 8, 4, 128)):
        cfg = P.ModelConfig(n_layers=1, n_heads=H, n_kv_heads=kvh, head_dim=dh, d_ff=dff, vocab_size=300, max_seq=1024)
        w = P.generate_weights(cfg, 502, tied_head=False)
        from tests.test_gpu_session import bf16_weights
        w = bf16_weights(P, w)
        om = O.OModel(O.OConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__}), O.round_weights_bf16(w.tensors), False)
        prompt = rng.integers(1, 300, 314).tolist()
        dc, oc = P.FullCache.from_config(cfg), O.OFullCache(1, kvh, dh, 1024, kv_bf16=True)
        g = P.prefill(w, prompt, dc)
        r = O.prefill(om, prompt, oc)
        gk = dc.k[0, :, :314].permute(1, 0, 2).float().cpu().numpy()
        ok = oc.rows[0].k
        mism = (gk != ok).mean()
        print(f"1-layer prefill dh{dh} H{H}: K mismatch fraction {mism:.3g}, max |dK| {np.abs(gk - ok).max():.3g}; "
              f"logits rel err {np.abs(g - r).max() / np.abs(r).max():.3g}", flush=True)


if __name__ == "__main__":
    main()
