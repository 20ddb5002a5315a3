"""Imported HF checkpoints on the device (`-m gpu`): the tensor-by-tensor
bf16 packing of checkpoint.load_hf_llama(device=True) equals the packing of
the host import, and forwards / a hierarchical session over imported weights
(YaRN rope table, head_dim 128 -> the tcgen05 attention) match the oracle."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2404_11912_b200 as pkg
    from paper_2404_11912_b200 import checkpoint
    return pkg, checkpoint


def _write(P, ck, path, cfg, seed, tied, scaling):
    w = P.generate_weights(cfg, seed, tied_head=tied)
    ck.save_hf_llama(w, path, dtype="BF16", rope_scaling=scaling, shard_bytes=8 << 20)
    return path


def test_hf_checkpoint_device_packing_and_forward(P, tmp_path):
    from oracle import hs_oracle as O
    P, ck = P
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=128, d_ff=688, vocab_size=300, max_seq=2048)
    yarn = ck.RopeScaling("yarn", 4.0, original_max_position_embeddings=512)
    d = _write(P, ck, tmp_path / "t", cfg, 3, False, yarn)
    host = ck.load_hf_llama(d)
    dev = ck.load_hf_llama(d, device=True)
    a, b = host.device(), dev.device()
    for name in ("wqkv", "wo", "wgu", "wdown", "emb", "head", "attn_norm", "mlp_norm", "final_norm",
                 "rope_cos", "rope_sin"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    c, s = yarn.tables(cfg.max_seq, cfg.head_dim, cfg.rope_theta)
    assert torch.equal(b.rope_cos.cpu(), torch.from_numpy(c))

    prompt = np.random.default_rng(4).integers(1, 256, 700).tolist()
    cache = P.FullCache.from_config(cfg)
    lg = P.prefill(dev, prompt, cache)
    rows = np.stack([P.decode_step(dev, t, cache) for t in (5, 9, 200)])

    ocfg = O.OConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
    om = O.OModel(ocfg, host.tensors, False)
    om.cos, om.sin = c.astype(np.float64), s.astype(np.float64)
    oc = O.OFullCache(cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, cfg.max_seq, kv_bf16=True)
    want = O.prefill(om, prompt, oc)
    want_rows = np.stack([O.decode_step(om, t, oc) for t in (5, 9, 200)])
    # same bar as test_forward_randomized_configs_match_oracle: fp32
    # accumulation differences occasionally flip the bf16 rounding of a cached
    # K/V entry, reaching ~3e-4 of the largest logit over 2 layers
    assert np.allclose(lg, want, rtol=1e-4, atol=1e-3 * np.abs(want).max())
    assert np.allclose(rows, want_rows, rtol=1e-4, atol=1e-3 * np.abs(want_rows).max())
    assert (np.argmax(lg, -1) == np.argmax(want, -1)).mean() > 0.99
    assert (np.argmax(rows, -1) == np.argmax(want_rows, -1)).all()


def test_hierarchical_session_on_imported_checkpoints(P, tmp_path):
    """Target and draft both imported (planted successor channel so the
    draft agrees often): greedy stream == autoregressive == oracle."""
    from oracle import hs_oracle as O
    P, ck = P
    tcfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=128, d_ff=688, vocab_size=260, max_seq=1024)
    dcfg = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=64, d_ff=172, vocab_size=260, max_seq=1024)
    tw = P.plant_successor(P.generate_weights(tcfg, 1, tied_head=False), 3, 0.9)
    dw = P.plant_successor(P.generate_weights(dcfg, 2, tied_head=False), 3, 0.9)
    ck.save_hf_llama(tw, tmp_path / "t", dtype="BF16")
    ck.save_hf_llama(dw, tmp_path / "d", dtype="BF16")
    ti, di = ck.load_hf_llama(tmp_path / "t", device=True), ck.load_hf_llama(tmp_path / "d", device=True)
    prompt = np.random.default_rng(0).integers(1, 256, 300).tolist()
    spec = P.SpecConfig(target_len=364, gamma1=2, gamma2=4, temperature=0.0, seed=0,
                        streaming=P.StreamingConfig(n_sink=4, budget=64),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=64, rebuild_stride=16))
    out, trace = P.HierarchicalSession(ti, di, prompt, spec).generate()
    assert out == P.autoregressive_generate(ti, prompt, 364, 0.0, 0)
    th = ck.load_hf_llama(tmp_path / "t")
    om = O.OModel(O.OConfig(**{k: getattr(tcfg, k) for k in tcfg.__dataclass_fields__}), th.tensors, False)
    assert out == O.ar_generate(om, prompt, 364, 0.0, 0, kv_bf16=True)
    assert trace.inner.accepted > 0 and trace.outer.accepted > 0
