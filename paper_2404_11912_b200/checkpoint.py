"""Real-checkpoint import: Hugging Face Llama safetensors -> this package's
weights (second half: "a safetensors import for real
checkpoints").  The reference reads only its own TFWT files
(hierspec/weights_io.py:31-95) and draws random weights
(hierspec/model.py:146-157); this module maps a `LlamaForCausalLM`
directory (Llama-2-7B/13B-128K, LWM-Text, JackFram/llama-68m ...) onto the
same tensor set (`model.tensor_order`, model.py:63-82), so a real target and
draft can sit beside the random-init ones in every session API.

Mapping (HF stores nn.Linear weights as [out][in]; the reference's layout is
x @ W with W [in][out]):

    model.embed_tokens.weight               [V, d]   -> embedding         (as is)
    model.layers.i.input_layernorm.weight   [d]      -> layers.i.attn_norm
    model.layers.i.self_attn.{q,k,v,o}_proj [out,in] -> layers.i.w{q,k,v,o} (transposed)
    model.layers.i.post_attention_layernorm [d]      -> layers.i.mlp_norm
    model.layers.i.mlp.{gate,up,down}_proj  [out,in] -> layers.i.w_{gate,up,down} (transposed)
    model.norm.weight                       [d]      -> final_norm
    lm_head.weight                          [V, d]   -> lm_head (transposed; absent when tied)

RoPE: the reference rotates interleaved pairs (2i, 2i+1) (model.py:235-244,
Meta's original layout); HF checkpoints are converted to the rotate-half
layout by permuting the rows of q_proj / k_proj inside each head
(`w.view(H, dh/2, 2, d).transpose(1, 2)`), so the import applies the inverse
permutation.  `rope_scaling` ("linear", "yarn", "llama3") is carried as a
`RopeScaling` next to the config; it changes only the cos/sin table the
kernels read (HF folds the YaRN attention factor into cos/sin the same way).

The safetensors container is parsed here directly (8-byte little-endian
header length, JSON header, raw little-endian payload); BF16 / F16 / F32
tensors are widened to fp32 exactly.  `device=True` packs each matrix into
the bf16 device layout tensor by tensor, never materialising a full fp32
host copy of a 7B/13B model.
"""

from __future__ import annotations

import json
import math
import os
import struct
from dataclasses import dataclass
from pathlib import Path
from typing import Callable, Dict, Optional, Tuple

import numpy as np

from .errors import ConfigError, TruncatedFileError, WeightFormatError
from .model import DeviceModel, ModelConfig, ModelWeights, tensor_order

_DTYPES = {"BF16": (np.uint16, 2), "F16": (np.float16, 2), "F32": (np.float32, 4)}


@dataclass(frozen=True)
class RopeScaling:
    """`rope_scaling` of a HF config, restated for the table build
    (transformers' _compute_{linear_scaling,yarn,llama3}_parameters)."""
    kind: str                               # "linear" | "yarn" | "llama3"
    factor: float
    original_max_position_embeddings: int = 0
    beta_fast: float = 32.0
    beta_slow: float = 1.0
    attention_factor: Optional[float] = None
    mscale: Optional[float] = None
    mscale_all_dim: Optional[float] = None
    truncate: bool = True
    low_freq_factor: float = 1.0
    high_freq_factor: float = 4.0

    @classmethod
    def from_hf(cls, d: Optional[dict], max_position_embeddings: int) -> Optional["RopeScaling"]:
        if not d:
            return None
        kind = d.get("rope_type", d.get("type", "default"))
        if kind == "default":
            return None
        if kind not in ("linear", "yarn", "llama3"):
            raise ConfigError(f"rope_scaling type {kind!r} is not supported (linear, yarn, llama3)")
        omax = int(d.get("original_max_position_embeddings") or 0)
        factor = d.get("factor")
        if factor is None:
            if kind != "yarn" or not omax:
                raise ConfigError(f"rope_scaling {kind!r} needs a factor")
            factor = max_position_embeddings / omax
        if kind in ("yarn", "llama3") and not omax:
            raise ConfigError(f"rope_scaling {kind!r} needs original_max_position_embeddings")
        return cls(kind=kind, factor=float(factor), original_max_position_embeddings=omax,
                   beta_fast=float(d.get("beta_fast") or 32.0), beta_slow=float(d.get("beta_slow") or 1.0),
                   attention_factor=d.get("attention_factor"), mscale=d.get("mscale"),
                   mscale_all_dim=d.get("mscale_all_dim"), truncate=bool(d.get("truncate", True)),
                   low_freq_factor=float(d.get("low_freq_factor", 1.0)),
                   high_freq_factor=float(d.get("high_freq_factor", 4.0)))

    def to_hf(self) -> dict:
        d = {"rope_type": self.kind, "factor": self.factor}
        if self.kind in ("yarn", "llama3"):
            d["original_max_position_embeddings"] = self.original_max_position_embeddings
        if self.kind == "yarn":
            d.update(beta_fast=self.beta_fast, beta_slow=self.beta_slow, truncate=self.truncate)
            for k in ("attention_factor", "mscale", "mscale_all_dim"):
                if getattr(self, k) is not None:
                    d[k] = getattr(self, k)
        if self.kind == "llama3":
            d.update(low_freq_factor=self.low_freq_factor, high_freq_factor=self.high_freq_factor)
        return d

    def inv_freq(self, head_dim: int, theta: float) -> Tuple[np.ndarray, float]:
        """(fp64 inverse frequencies [head_dim/2], cos/sin multiplier)."""
        dim = head_dim
        base = np.power(np.float64(theta), np.arange(0, dim, 2, dtype=np.float64) / np.float64(dim))
        inv = 1.0 / base
        if self.kind == "linear":
            return inv / self.factor, 1.0
        if self.kind == "llama3":
            old = self.original_max_position_embeddings
            lo_w, hi_w = old / self.low_freq_factor, old / self.high_freq_factor
            wav = 2 * math.pi / inv
            out = np.where(wav > lo_w, inv / self.factor, inv)
            smooth = (old / wav - self.low_freq_factor) / (self.high_freq_factor - self.low_freq_factor)
            smoothed = (1 - smooth) * out / self.factor + smooth * out
            medium = ~(wav < hi_w) & ~(wav > lo_w)
            return np.where(medium, smoothed, out), 1.0
        # yarn
        def mscale(s, m=1.0):
            return 1.0 if s <= 1 else 0.1 * m * math.log(s) + 1.0
        att = self.attention_factor
        if att is None:
            att = (mscale(self.factor, self.mscale) / mscale(self.factor, self.mscale_all_dim)
                   if self.mscale and self.mscale_all_dim else mscale(self.factor))

        def corr_dim(rot):
            return dim * math.log(self.original_max_position_embeddings / (rot * 2 * math.pi)) / (2 * math.log(theta))
        lo, hi = corr_dim(self.beta_fast), corr_dim(self.beta_slow)
        if self.truncate:
            lo, hi = math.floor(lo), math.ceil(hi)
        lo, hi = max(lo, 0), min(hi, dim - 1)
        if lo == hi:
            hi += 0.001
        ramp = np.clip((np.arange(dim // 2, dtype=np.float64) - lo) / (hi - lo), 0.0, 1.0)
        extra = 1.0 - ramp
        return (inv / self.factor) * (1.0 - extra) + inv * extra, float(att)

    def tables(self, n_pos: int, head_dim: int, theta: float) -> Tuple[np.ndarray, np.ndarray]:
        """fp32 cos/sin [n_pos, head_dim/2]: fp64 angles (and factor), rounded
        once to fp32 like model.rope_tables (tensor.py:66-76)."""
        inv, att = self.inv_freq(head_dim, theta)
        ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
        return (np.cos(ang) * att).astype(np.float32), (np.sin(ang) * att).astype(np.float32)


# ----------------------------------------------------------------------------- safetensors container

class SafetensorsFile:
    """Lazy reader of one .safetensors file (memory-mapped)."""

    def __init__(self, path):
        self.path = str(path)
        self._mm = np.memmap(self.path, dtype=np.uint8, mode="r")
        if self._mm.size < 8:
            raise TruncatedFileError(f"{path}: shorter than the 8-byte header length")
        (hlen,) = struct.unpack("<Q", self._mm[:8].tobytes())
        if 8 + hlen > self._mm.size:
            raise TruncatedFileError(f"{path}: header of {hlen} bytes past the end of the file")
        try:
            header = json.loads(self._mm[8:8 + hlen].tobytes())
        except ValueError as e:
            raise WeightFormatError(f"{path}: bad safetensors header: {e}") from None
        self.metadata = header.pop("__metadata__", {})
        self.base = 8 + hlen
        self.entries = header
        for name, e in header.items():
            if e.get("dtype") not in _DTYPES:
                raise WeightFormatError(f"{path}: {name}: dtype {e.get('dtype')} not supported (BF16/F16/F32)")
            a, b = e["data_offsets"]
            n = int(np.prod(e["shape"])) if e["shape"] else 1
            if b - a != n * _DTYPES[e["dtype"]][1] or self.base + b > self._mm.size:
                raise WeightFormatError(f"{path}: {name}: data_offsets {a}:{b} do not hold shape {e['shape']}")

    def raw(self, name: str) -> Tuple[str, np.ndarray]:
        """(dtype string, array view with the stored element type)."""
        e = self.entries[name]
        a, b = e["data_offsets"]
        np_t, _ = _DTYPES[e["dtype"]]
        return e["dtype"], self._mm[self.base + a:self.base + b].view(np_t).reshape(e["shape"])

    def f32(self, name: str) -> np.ndarray:
        """Tensor widened exactly to fp32."""
        dt, a = self.raw(name)
        if dt == "BF16":
            return (a.astype(np.uint32) << 16).view(np.float32)
        return a.astype(np.float32)


def _open_dir(path) -> Tuple[dict, Dict[str, SafetensorsFile]]:
    """(config.json dict, tensor name -> file) for a HF model directory (or one
    .safetensors file with a config.json beside it)."""
    p = Path(path)
    d = p if p.is_dir() else p.parent
    cfg_path = d / "config.json"
    if not cfg_path.exists():
        raise WeightFormatError(f"{d}: no config.json")
    hf = json.loads(cfg_path.read_text())
    if p.is_file():
        files = [p]
    elif (d / "model.safetensors.index.json").exists():
        idx = json.loads((d / "model.safetensors.index.json").read_text())
        files = sorted({d / f for f in idx["weight_map"].values()})
    else:
        files = sorted(d.glob("*.safetensors"))
    if not files:
        raise WeightFormatError(f"{d}: no .safetensors files")
    where = {}
    for f in files:
        sf = SafetensorsFile(f)
        for name in sf.entries:
            where[name] = sf
    return hf, where


def hf_config(hf: dict, max_seq: Optional[int] = None) -> Tuple[ModelConfig, bool, Optional[RopeScaling]]:
    """ModelConfig, tied-head flag and rope scaling of a HF Llama config.json."""
    arch = hf.get("architectures") or ["LlamaForCausalLM"]
    if hf.get("model_type", "llama") not in ("llama", "mistral") and "LlamaForCausalLM" not in arch:
        raise ConfigError(f"not a Llama checkpoint: model_type {hf.get('model_type')!r}")
    if hf.get("hidden_act", "silu") != "silu":
        raise ConfigError(f"hidden_act {hf.get('hidden_act')!r}: the dense path is SwiGLU (model.py:322)")
    if hf.get("attention_bias") or hf.get("mlp_bias"):
        raise ConfigError("projection biases are not part of the reference architecture")
    d, H = int(hf["hidden_size"]), int(hf["num_attention_heads"])
    dh = int(hf.get("head_dim") or d // H)
    if dh * H != d:
        raise ConfigError(f"head_dim {dh} x {H} heads != hidden_size {d}")
    mpe = int(hf.get("max_position_embeddings", 2048))
    rp = hf.get("rope_parameters") or {}
    theta = float(hf.get("rope_theta", rp.get("rope_theta", 10000.0)))
    scaling = RopeScaling.from_hf(hf.get("rope_scaling") or (rp if rp.get("rope_type", "default") != "default"
                                                             else None), mpe)
    cfg = ModelConfig(n_layers=int(hf["num_hidden_layers"]), n_heads=H,
                      n_kv_heads=int(hf.get("num_key_value_heads") or H), head_dim=dh,
                      d_ff=int(hf["intermediate_size"]), vocab_size=int(hf["vocab_size"]),
                      max_seq=int(max_seq or mpe), rope_theta=theta, norm_eps=float(hf.get("rms_norm_eps", 1e-6)))
    return cfg, bool(hf.get("tie_word_embeddings", False)), scaling


def _unpermute(w: np.ndarray, heads: int) -> np.ndarray:
    """HF rotate-half row order -> interleaved pairs, rows of one projection
    [heads*dh, in]: row p*dh/2 + i of a head becomes row 2i + p."""
    out_dim, k = w.shape
    dh = out_dim // heads
    return w.reshape(heads, 2, dh // 2, k).transpose(0, 2, 1, 3).reshape(out_dim, k)


def _permute(w: np.ndarray, heads: int) -> np.ndarray:
    """Interleaved pairs -> HF rotate-half rows (the HF conversion script's permute)."""
    out_dim, k = w.shape
    dh = out_dim // heads
    return w.reshape(heads, dh // 2, 2, k).transpose(0, 2, 1, 3).reshape(out_dim, k)


def _hf_names(cfg: ModelConfig, tied: bool):
    """(our name, HF name, transpose, q/k head count for the row permutation)."""
    out = [("embedding", "model.embed_tokens.weight", False, 0)]
    for i in range(cfg.n_layers):
        p = f"model.layers.{i}."
        out += [(f"layers.{i}.attn_norm", p + "input_layernorm.weight", False, 0),
                (f"layers.{i}.wq", p + "self_attn.q_proj.weight", True, cfg.n_heads),
                (f"layers.{i}.wk", p + "self_attn.k_proj.weight", True, cfg.n_kv_heads),
                (f"layers.{i}.wv", p + "self_attn.v_proj.weight", True, 0),
                (f"layers.{i}.wo", p + "self_attn.o_proj.weight", True, 0),
                (f"layers.{i}.mlp_norm", p + "post_attention_layernorm.weight", False, 0),
                (f"layers.{i}.w_gate", p + "mlp.gate_proj.weight", True, 0),
                (f"layers.{i}.w_up", p + "mlp.up_proj.weight", True, 0),
                (f"layers.{i}.w_down", p + "mlp.down_proj.weight", True, 0)]
    out.append(("final_norm", "model.norm.weight", False, 0))
    if not tied:
        out.append(("lm_head", "lm_head.weight", True, 0))
    return out


def load_hf_llama(path, device: bool = False, max_seq: Optional[int] = None) -> ModelWeights:
    """Load a HF Llama safetensors checkpoint (directory with config.json).

    device=False: host fp32 `ModelWeights` in the reference layout (exact
    widening of BF16/F16/F32).  device=True: a device-only `ModelWeights`
    whose bf16 packing is filled tensor by tensor (the 7B/13B case).
    max_seq overrides max_position_embeddings (the rope table length).
    Raises WeightFormatError for a missing / mis-shaped tensor and ConfigError
    for architectures the reference's forward does not compute.
    """
    hf, where = _open_dir(path)
    cfg, tied, scaling = hf_config(hf, max_seq)
    if not tied and "lm_head.weight" not in where:
        tied = True                                  # HF omits the head of tied checkpoints
    expected = dict(tensor_order(cfg, tied))

    def fetch(ours: str, name: str, transpose: bool, heads: int, widen: Callable) -> np.ndarray:
        if name not in where:
            raise WeightFormatError(f"{path}: tensor {name} missing")
        a = widen(where[name], name)
        if heads:
            a = _unpermute(a, heads)
        if transpose:
            a = a.T
        if tuple(a.shape) != expected[ours]:
            raise WeightFormatError(f"{path}: {name} has shape {a.shape[::-1] if transpose else a.shape}, "
                                    f"config implies {expected[ours]}")
        return a

    names = _hf_names(cfg, tied)
    if not device:
        tensors = {ours: np.ascontiguousarray(fetch(ours, n, tr, h, lambda f, k: f.f32(k)))
                   for ours, n, tr, h in names}
        return ModelWeights(cfg, tensors, tied, rope_scaling=scaling).validate()

    def bf16_rows(ours, n, tr, h) -> np.ndarray:      # [out][in] fp32 view for the device packer
        return fetch(ours, n, tr, h, lambda f, k: f.f32(k))
    dm = DeviceModel.from_tensor_source(cfg, tied, lambda ours: _lookup(names, ours, bf16_rows),
                                        rope_scaling=scaling)
    return ModelWeights.on_device(dm)


def _lookup(names, ours, fn):
    for row in names:
        if row[0] == ours:
            return fn(*row)
    raise KeyError(ours)


def save_hf_llama(weights: ModelWeights, path, dtype: str = "F32", rope_scaling: Optional[RopeScaling] = None,
                  shard_bytes: Optional[int] = None) -> None:
    """Write `weights` as a HF Llama directory (config.json + safetensors,
    rotate-half q/k rows).  F32 round trips bit-exactly; BF16 rounds to
    nearest even.  shard_bytes splits the tensors over several files with a
    model.safetensors.index.json, as large HF checkpoints are laid out."""
    if dtype not in ("F32", "BF16"):
        raise ValueError("dtype must be F32 or BF16")
    weights.validate()
    cfg, tied = weights.config, weights.tied_head
    d = Path(path)
    d.mkdir(parents=True, exist_ok=True)
    scaling = rope_scaling if rope_scaling is not None else getattr(weights, "rope_scaling", None)
    hf = {"architectures": ["LlamaForCausalLM"], "model_type": "llama", "hidden_size": cfg.d_model,
          "num_attention_heads": cfg.n_heads, "num_key_value_heads": cfg.n_kv_heads, "head_dim": cfg.head_dim,
          "intermediate_size": cfg.d_ff, "num_hidden_layers": cfg.n_layers, "vocab_size": cfg.vocab_size,
          "max_position_embeddings": cfg.max_seq, "rope_theta": cfg.rope_theta, "rms_norm_eps": cfg.norm_eps,
          "tie_word_embeddings": tied, "hidden_act": "silu", "attention_bias": False, "mlp_bias": False,
          "torch_dtype": "float32" if dtype == "F32" else "bfloat16", "rope_scaling": scaling.to_hf() if scaling else None}
    (d / "config.json").write_text(json.dumps(hf, indent=1))
    blobs = []
    for ours, name, tr, heads in _hf_names(cfg, tied):
        a = np.asarray(weights.tensors[ours], dtype=np.float32)
        if tr:
            a = a.T
        if heads:
            a = _permute(np.ascontiguousarray(a), heads)
        a = np.ascontiguousarray(a)
        if dtype == "BF16":
            u = a.view(np.uint32).astype(np.uint64)
            u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16        # round to nearest even
            raw = u.astype(np.uint16).tobytes()
        else:
            raw = a.astype("<f4").tobytes()
        blobs.append((name, list(a.shape), raw))
    groups, cur, size = [], [], 0
    for b in blobs:
        if shard_bytes and cur and size + len(b[2]) > shard_bytes:
            groups.append(cur)
            cur, size = [], 0
        cur.append(b)
        size += len(b[2])
    groups.append(cur)
    wmap = {}
    for gi, grp in enumerate(groups):
        fname = "model.safetensors" if len(groups) == 1 else f"model-{gi + 1:05d}-of-{len(groups):05d}.safetensors"
        header, off = {}, 0
        for name, shape, raw in grp:
            header[name] = {"dtype": dtype, "shape": shape, "data_offsets": [off, off + len(raw)]}
            off += len(raw)
            wmap[name] = fname
        hj = json.dumps(header).encode()
        hj += b" " * (-len(hj) % 8)
        with open(d / fname, "wb") as f:
            f.write(struct.pack("<Q", len(hj)))
            f.write(hj)
            for _, _, raw in grp:
                f.write(raw)
    if len(groups) > 1:
        (d / "model.safetensors.index.json").write_text(json.dumps({"metadata": {}, "weight_map": wmap}))
