"""HF Llama safetensors import (checkpoint.py).

The oracle (oracle/hs_oracle.py, the reference's forward restated) run on the
imported weights must match transformers' own LlamaForCausalLM forward on
the same checkpoint: that pins the name mapping, the [out][in] transposes,
the q/k rotate-half -> interleaved row permutation and the rope-scaling
tables against an independent implementation.  CPU only; the device packing
is covered in test_gpu_kernels.py::test_hf_checkpoint_device_packing.
"""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

from oracle import hs_oracle as O


@pytest.fixture(scope="module")
def M():
    from paper_2404_11912_b200 import checkpoint, errors, model
    return model, checkpoint, errors


def _cfg(model, **kw):
    base = dict(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=16, d_ff=96, vocab_size=80, max_seq=256)
    base.update(kw)
    return model.ModelConfig(**base)


def test_round_trip_f32_bitwise(M, tmp_path):
    model, ck, _ = M
    for tied, shard in ((False, None), (True, None), (False, 40_000)):
        w = model.generate_weights(_cfg(model), 5, tied_head=tied)
        d = tmp_path / f"rt_{tied}_{shard}"
        ck.save_hf_llama(w, d, shard_bytes=shard)
        if shard:
            assert (d / "model.safetensors.index.json").exists()
        back = ck.load_hf_llama(d)
        assert back.config == w.config and back.tied_head == tied
        for k in w.tensors:
            assert np.array_equal(back.tensors[k].view(np.uint32), w.tensors[k].view(np.uint32)), k


def test_bf16_is_round_to_nearest_even(M, tmp_path):
    model, ck, _ = M
    w = model.generate_weights(_cfg(model), 6, tied_head=False)
    ck.save_hf_llama(w, tmp_path / "b", dtype="BF16")
    back = ck.load_hf_llama(tmp_path / "b")
    for k in w.tensors:
        want = torch.from_numpy(w.tensors[k]).to(torch.bfloat16).float().numpy()
        assert np.array_equal(back.tensors[k], want), k


def _oracle_logits(w, tokens, scaling=None):
    cfg = O.OConfig(**{k: getattr(w.config, k) for k in w.config.__dataclass_fields__})
    om = O.OModel(cfg, w.tensors, w.tied_head)
    if scaling is not None:
        c, s = scaling.tables(cfg.max_seq, cfg.head_dim, cfg.rope_theta)
        om.cos, om.sin = c.astype(np.float64), s.astype(np.float64)
    cache = O.OFullCache(cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, cfg.max_seq)
    return O.prefill(om, tokens, cache)


def _hf_model(tmp_path, name, rope_scaling=None, tied=False, kvh=2):
    from transformers import LlamaConfig, LlamaForCausalLM
    torch.manual_seed(0)
    kw = dict(vocab_size=80, hidden_size=64, intermediate_size=96, num_hidden_layers=2, num_attention_heads=4,
              num_key_value_heads=kvh, max_position_embeddings=256, rms_norm_eps=1e-5, rope_theta=10000.0,
              tie_word_embeddings=tied, attention_bias=False)
    if rope_scaling is not None:
        kw["rope_scaling"] = rope_scaling
    hf = LlamaForCausalLM(LlamaConfig(**kw)).float().eval()
    with torch.no_grad():                     # non-trivial norm gains (HF initialises them to 1)
        for n, p in hf.named_parameters():
            if "norm" in n:
                p.add_(torch.randn_like(p) * 0.1)
    d = tmp_path / name
    hf.save_pretrained(d, safe_serialization=True)
    return hf, d


@pytest.mark.parametrize("rope", [None, {"rope_type": "linear", "factor": 4.0},
                                  {"rope_type": "yarn", "factor": 8.0, "original_max_position_embeddings": 32},
                                  {"rope_type": "llama3", "factor": 8.0, "low_freq_factor": 1.0,
                                   "high_freq_factor": 4.0, "original_max_position_embeddings": 32}],
                         ids=["plain", "linear", "yarn", "llama3"])
def test_oracle_on_import_matches_transformers(M, tmp_path, rope):
    _, ck, _ = M
    hf, d = _hf_model(tmp_path, "hf", rope)
    w = ck.load_hf_llama(d)
    assert (w.rope_scaling is None) == (rope is None)
    tokens = np.random.default_rng(1).integers(0, 80, 200).tolist()
    with torch.no_grad():
        want = hf(torch.tensor([tokens])).logits[0].double().numpy()
    got = _oracle_logits(w, tokens, w.rope_scaling)
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err < 2e-5, err
    if rope is not None:       # the table's frequencies are HF's (fp64 vs HF's fp32 evaluation)
        inv, att = w.rope_scaling.inv_freq(16, 10000.0)
        rot = hf.model.rotary_emb
        np.testing.assert_allclose(inv, rot.inv_freq.double().numpy(), rtol=1e-6)
        assert abs(att - float(rot.attention_scaling)) < 1e-6


def test_tied_and_mha_checkpoints(M, tmp_path):
    _, ck, _ = M
    hf, d = _hf_model(tmp_path, "tied", tied=True, kvh=4)
    w = ck.load_hf_llama(d)
    assert w.tied_head and w.config.n_kv_heads == 4
    tokens = list(range(3, 70))
    with torch.no_grad():
        want = hf(torch.tensor([tokens])).logits[0].double().numpy()
    got = _oracle_logits(w, tokens)
    assert np.abs(got - want).max() / np.abs(want).max() < 2e-5


def test_import_errors(M, tmp_path):
    model, ck, err = M
    w = model.generate_weights(_cfg(model), 7, tied_head=False)
    d = tmp_path / "e"
    ck.save_hf_llama(w, d)
    cfg = json.loads((d / "config.json").read_text())
    cfg["rope_scaling"] = {"rope_type": "dynamic", "factor": 2.0}
    (d / "config.json").write_text(json.dumps(cfg))
    with pytest.raises(err.ConfigError):
        ck.load_hf_llama(d)
    cfg["rope_scaling"] = None
    cfg["intermediate_size"] = 97
    (d / "config.json").write_text(json.dumps(cfg))
    with pytest.raises(err.WeightFormatError):
        ck.load_hf_llama(d)
    cfg["intermediate_size"] = 96
    (d / "config.json").write_text(json.dumps(cfg))
    raw = (d / "model.safetensors").read_bytes()
    (d / "model.safetensors").write_bytes(raw[:-4])
    with pytest.raises(err.WeightFormatError):
        ck.load_hf_llama(d)
    (d / "model.safetensors").write_bytes(raw[:6])
    with pytest.raises(err.TruncatedFileError):
        ck.load_hf_llama(d)
    with pytest.raises(err.WeightFormatError):
        ck.load_hf_llama(tmp_path / "nowhere")
    from paper_2404_11912_b200 import weights_io
    with pytest.raises(err.WeightFormatError):        # TFWT cannot carry rope scaling
        weights_io.save_weights(model.ModelWeights(w.config, w.tensors, False,
                                                   rope_scaling=ck.RopeScaling("linear", 2.0)), tmp_path / "x")
