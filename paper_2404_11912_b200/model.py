"""Decoder-only Llama block on B200: model config, weights, forward entry
points and sampling -- the drop-in for hierspec/model.py.

Same names, signatures and error behaviour as the reference
(model.py:28-393); the arithmetic runs in the sm_100a library:

* weights are packed once per device to bf16 [out][in] (`DeviceModel`,
  replacing `ModelWeights.runtime()`, model.py:116-143);
* `prefill` / `decode_step` / `decode_chunk` call `hs_forward`, one native
  call per lane step; `decode_chunk` is a single batched forward whose rows
  are bit-identical to a `decode_step` loop (the kernels' reductions do not
  depend on the batch size), which is the reference's own contract
  (model.py:366-378) -- except over a TopKCache, whose per-query selection
  makes the chunk a loop of single-token forwards, as in the reference;
* sampling (`prob_from_logits`, `sample_from_probs`) runs in fp64 kernels
  consuming exactly one uniform per draw from the caller's Generator.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _abi
from ._abi import HsModel, check, lib
from .errors import CapacityError, ContractError, FiniteError, ShapeError
from .runtime import STATS, as_device_f32, as_device_f64, device, ptr, stream_ptr, to_i32_device, workspaces

BOS = 256
EOS = 257
PAD = 258
TOKENIZER_VOCAB = 259


# projection matrices stored tile-blocked on the device (HsModel.blocked): every
# 128 x 64 GEMV / GEMM tile one contiguous 16 KB block, so a CTA's weight stream
# is sequential in HBM (HS_ROWMAJOR_WEIGHTS=1: row-major, an A/B hook)
BLOCK_WEIGHTS = os.environ.get("HS_ROWMAJOR_WEIGHTS", "0") != "1"


def _pad64(n: int) -> int:
    return (n + 63) // 64 * 64


@dataclass(frozen=True)
class ModelConfig:
    """Architecture hyper-parameters (model.py:28-59)."""
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab_size: int
    max_seq: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    def __post_init__(self):
        for name in ("n_layers", "n_heads", "n_kv_heads", "head_dim", "d_ff"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be positive")
        if self.n_heads % self.n_kv_heads:
            raise ValueError("n_heads must be a multiple of n_kv_heads")
        if self.head_dim % 2:
            raise ValueError("head_dim must be even")
        if self.max_seq < 1 or self.vocab_size < 2:
            raise ValueError("max_seq >= 1 and vocab_size >= 2 required")
        # reals live as f32 in the weight format: canonicalise (model.py:50-53)
        object.__setattr__(self, "rope_theta", float(np.float32(self.rope_theta)))
        object.__setattr__(self, "norm_eps", float(np.float32(self.norm_eps)))
        if self.rope_theta <= 0 or self.norm_eps < 0:
            raise ValueError("rope_theta must be positive and norm_eps non-negative")

    @property
    def d_model(self) -> int:
        return self.n_heads * self.head_dim


def tensor_order(config: ModelConfig, tied_head: bool):
    """Weight tensor names and shapes in file/generation order (model.py:63-82)."""
    d, kv = config.d_model, config.n_kv_heads * config.head_dim
    names = [("embedding", (config.vocab_size, d))]
    for i in range(config.n_layers):
        for suffix, shape in (("attn_norm", (d,)), ("wq", (d, d)), ("wk", (d, kv)), ("wv", (d, kv)),
                              ("wo", (d, d)), ("mlp_norm", (d,)), ("w_gate", (d, config.d_ff)),
                              ("w_up", (d, config.d_ff)), ("w_down", (config.d_ff, d))):
            names.append((f"layers.{i}.{suffix}", shape))
    names.append(("final_norm", (d,)))
    if not tied_head:
        names.append(("lm_head", (d, config.vocab_size)))
    return names


def rope_tables(n_pos: int, head_dim: int, theta: float):
    """fp32 cos/sin [n_pos, head_dim/2]: fp64 angles rounded once to fp32
    (tensor.py:66-76)."""
    half = head_dim // 2
    inv = np.power(np.float64(theta), -2.0 * np.arange(half, dtype=np.float64) / np.float64(head_dim))
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


class DeviceModel:
    """bf16 packing of a model on one CUDA device plus its `HsModel` descriptor.

    Layout (include/hs_abi.h): matrices transposed to [out][in] with the row
    stride padded to 64 elements; wq|wk|wv fused; gate/up rows interleaved
    (gate_i, up_i) so the GEMV's SwiGLU epilogue sees both halves; norms and
    the rope table stay fp32.  When every projection has a multiple of 128
    rows the projections (and an untied lm_head) are then stored tile-blocked
    ([N/128][ld/64][128][64], `blocked`): each 128 x 64 weight tile a GEMV or
    GEMM CTA streams is one contiguous 16 KB block.
    """

    def __init__(self, config: ModelConfig, tensors, tied_head: bool, rope_scaling=None):
        """tensors: name -> numpy [in, out] fp32 (the reference layout), as a
        dict or a callable fetching one tensor at a time (checkpoint import:
        only one matrix is on the host at once)."""
        self.config = config
        self.tied_head = tied_head
        self.rope_scaling = rope_scaling
        get = tensors if callable(tensors) else tensors.__getitem__
        dev = device()
        L, d, dff, V = config.n_layers, config.d_model, config.d_ff, config.vocab_size
        kv = config.n_kv_heads * config.head_dim
        self.ld_d, self.ld_ff = _pad64(d), _pad64(dff)
        nqkv = d + 2 * kv

        def mat(a, ld):   # numpy [in, out] fp32 -> torch [out, ld] bf16
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev).t()
            out = torch.zeros((t.shape[0], ld), dtype=torch.bfloat16, device=dev)
            out[:, :t.shape[1]] = t.to(torch.bfloat16)
            return out

        g = lambda i, n: get(f"layers.{i}.{n}")
        self.wqkv = torch.empty((L, nqkv, self.ld_d), dtype=torch.bfloat16, device=dev)
        self.wo = torch.empty((L, d, self.ld_d), dtype=torch.bfloat16, device=dev)
        self.wgu = torch.empty((L, 2 * dff, self.ld_d), dtype=torch.bfloat16, device=dev)
        self.wdown = torch.empty((L, d, self.ld_ff), dtype=torch.bfloat16, device=dev)
        self.attn_norm = torch.empty((L, d), dtype=torch.float32, device=dev)
        self.mlp_norm = torch.empty((L, d), dtype=torch.float32, device=dev)
        for i in range(L):
            self.wqkv[i] = mat(np.concatenate([g(i, "wq"), g(i, "wk"), g(i, "wv")], axis=1), self.ld_d)
            self.wo[i] = mat(g(i, "wo"), self.ld_d)
            gu = np.empty((d, 2 * dff), np.float32)
            gu[:, 0::2] = g(i, "w_gate")
            gu[:, 1::2] = g(i, "w_up")
            self.wgu[i] = mat(gu, self.ld_d)
            self.wdown[i] = mat(g(i, "w_down"), self.ld_ff)
            self.attn_norm[i] = torch.from_numpy(g(i, "attn_norm").astype(np.float32))
            self.mlp_norm[i] = torch.from_numpy(g(i, "mlp_norm").astype(np.float32))
        self.emb = mat(get("embedding").T, self.ld_d)
        self.head = self.emb if tied_head else mat(get("lm_head"), self.ld_d)
        self.final_norm = torch.from_numpy(get("final_norm").astype(np.float32)).to(dev)
        self._finish()

    @classmethod
    def from_tensor_source(cls, config: ModelConfig, tied_head: bool, get, rope_scaling=None) -> "DeviceModel":
        """Pack from a per-tensor getter (checkpoint.load_hf_llama)."""
        return cls(config, get, tied_head, rope_scaling)

    @classmethod
    def random(cls, config: ModelConfig, seed: int, tied_head: bool = False, std: float = 0.02):
        """Random-init weights generated directly on the device (bf16), for
        model sizes whose host fp32 copy is impractical (Llama2-7B shape).
        Same distribution as generate_weights, different stream."""
        self = cls.__new__(cls)
        self.config, self.tied_head, self.rope_scaling = config, tied_head, None
        dev = device()
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        L, d, dff, V = config.n_layers, config.d_model, config.d_ff, config.vocab_size
        kv = config.n_kv_heads * config.head_dim
        self.ld_d, self.ld_ff = _pad64(d), _pad64(dff)

        def rnd(rows, cols, ld):
            out = torch.zeros((rows, ld), dtype=torch.bfloat16, device=dev)
            out[:, :cols] = (torch.randn((rows, cols), generator=gen, device=dev) * std).to(torch.bfloat16)
            return out

        self.wqkv = torch.stack([rnd(d + 2 * kv, d, self.ld_d) for _ in range(L)])
        self.wo = torch.stack([rnd(d, d, self.ld_d) for _ in range(L)])
        self.wgu = torch.empty((L, 2 * dff, self.ld_d), dtype=torch.bfloat16, device=dev)
        for i in range(L):
            self.wgu[i] = rnd(2 * dff, d, self.ld_d)
        self.wdown = torch.stack([rnd(d, dff, self.ld_ff) for _ in range(L)])
        self.attn_norm = 1.0 + torch.randn((L, d), generator=gen, device=dev) * std
        self.mlp_norm = 1.0 + torch.randn((L, d), generator=gen, device=dev) * std
        self.emb = rnd(V, d, self.ld_d)
        self.head = self.emb if tied_head else rnd(V, d, self.ld_d)
        self.final_norm = 1.0 + torch.randn((d,), generator=gen, device=dev) * std
        self._finish()
        return self

    def plant_successor_(self, seed: int, easy_frac: float, emb_scale: float = 32.0, margin: float = 24.0):
        """Device-side `plant_successor` (same construction, torch RNG): for
        the easy tokens t, emb[t] += emb_scale * u_t and head[succ(t)] +=
        (margin / d) * u_t with u_t a random +-1 vector.  See plant_successor."""
        cfg = self.config
        V, d = cfg.vocab_size, cfg.d_model
        head_scale = margin / d
        dev = self.emb.device
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        succ = torch.randperm(V, generator=gen, device=dev)
        easy = torch.rand(V, generator=gen, device=dev) < easy_frac
        idx = torch.nonzero(easy).flatten()
        for a in range(0, idx.numel(), 4096):
            rows = idx[a:a + 4096]
            u = torch.randint(0, 2, (rows.numel(), d), generator=gen, device=dev).float() * 2.0 - 1.0
            self.emb[rows, :d] = (self.emb[rows, :d].float() + emb_scale * u).to(torch.bfloat16)
            hr = succ[rows]
            self._set_head_rows(hr, (self._head_rows(hr)[:, :d].float() + head_scale * u).to(torch.bfloat16))
        self.planted = {"kind": "successor", "easy_frac": easy_frac, "seed": seed, "emb_scale": emb_scale,
                        "margin": margin}
        return self

    def _head_rows(self, rows: torch.Tensor) -> torch.Tensor:
        """Rows of the lm_head [n, ld] whatever its device layout."""
        if not (getattr(self, "blocked", 0) & 2):
            return self.head[rows]
        ld = self.ld_d
        hv = self.head.view(-1, ld // 64, 128, 64)
        return hv[rows // 128, :, rows % 128, :].reshape(rows.numel(), ld)

    def _set_head_rows(self, rows: torch.Tensor, vals: torch.Tensor) -> None:
        """head[rows, :vals.shape[1]] = vals, whatever its device layout."""
        if not (getattr(self, "blocked", 0) & 2):
            self.head[rows, :vals.shape[1]] = vals
            return
        full = self._head_rows(rows)
        full[:, :vals.shape[1]] = vals
        ld = self.ld_d
        hv = self.head.view(-1, ld // 64, 128, 64)
        hv[rows // 128, :, rows % 128, :] = full.view(rows.numel(), ld // 64, 64)

    def _block_weights(self) -> int:
        """Re-lay the projection matrices (and an untied lm_head) tile-blocked
        in place (hs_weights_block); returns HsModel.blocked."""
        cfg = self.config
        kv = cfg.n_kv_heads * cfg.head_dim
        if not BLOCK_WEIGHTS or any(n % 128 for n in (cfg.d_model + 2 * kv, cfg.d_model, 2 * cfg.d_ff)):
            return 0
        mats = [self.wqkv, self.wo, self.wgu, self.wdown]
        head = not self.tied_head and cfg.vocab_size % 128 == 0
        n_tmp = max([m[0].numel() for m in mats] + ([self.head.numel()] if head else []))
        tmp = torch.empty(n_tmp, dtype=torch.bfloat16, device=self.wqkv.device)
        s = stream_ptr()
        for m in mats:
            for layer in range(m.shape[0]):
                check(lib.hs_weights_block(m[layer].data_ptr(), tmp.data_ptr(), m.shape[1], m.shape[2], 0, s))
        if head:
            check(lib.hs_weights_block(self.head.data_ptr(), tmp.data_ptr(), self.head.shape[0], self.head.shape[1],
                                       0, s))
        torch.cuda.current_stream().synchronize()   # (tmp is freed on return)
        return 1 | (2 if head else 0)

    def _finish(self):
        cfg = self.config
        scaling = getattr(self, "rope_scaling", None)
        cos, sin = (scaling.tables(cfg.max_seq, cfg.head_dim, cfg.rope_theta) if scaling is not None
                    else rope_tables(cfg.max_seq, cfg.head_dim, cfg.rope_theta))
        dev = device()
        self.rope_cos = torch.from_numpy(cos).to(dev)
        self.rope_sin = torch.from_numpy(sin).to(dev)
        s = HsModel()
        s.n_layers, s.n_heads, s.n_kv_heads = cfg.n_layers, cfg.n_heads, cfg.n_kv_heads
        s.head_dim, s.d_ff, s.vocab_size, s.max_seq = cfg.head_dim, cfg.d_ff, cfg.vocab_size, cfg.max_seq
        s.d_model, s.ld_d, s.ld_ff, s.norm_eps = cfg.d_model, self.ld_d, self.ld_ff, cfg.norm_eps
        for name in ("emb", "head", "final_norm", "attn_norm", "mlp_norm", "wqkv", "wo", "wgu", "wdown",
                     "rope_cos", "rope_sin"):
            setattr(s, name, getattr(self, name).data_ptr())
        self.blocked = self._block_weights()
        s.blocked = self.blocked
        self.struct = s
        self.ref = C.byref(s)

    def workspace(self, nbytes: int) -> torch.Tensor:
        """This model's forward workspace on the current stream.  Its head
        (GEMV arrival counters and K-split partials,
        hs_forward_workspace_clean_bytes) must be zero before first use and is
        left zero by every call; the layout of that head depends on the
        model's matrix shapes, so the buffer is owned by the model and never
        shared with another one -- nor between streams (the ranks of a
        loopback shard group run one model concurrently)."""
        if not hasattr(self, "_ws"):
            self._ws = {}
        key = stream_ptr()
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=self.emb.device)
            self._ws[key] = ws
        return ws

    def forward_ws_bytes(self, t: int, n_view: int, split: int, world: int) -> int:
        """hs_forward_workspace_bytes, memoised: it depends on n_view only
        through the number of attention splits."""
        key = (t, -(-n_view // split), split, world)
        memo = self.__dict__.setdefault("_ws_memo", {})
        nb = memo.get(key)
        if nb is None:
            nb = memo[key] = max(lib.hs_forward_workspace_bytes(self.ref, t, n_view, split, world),
                                 lib.hs_forward_workspace_bytes(self.ref, t, key[1] * split, split, world))
        return nb

    @property
    def weight_bytes(self) -> int:
        """Algorithmic weight bytes streamed per forward (embedding row excluded)."""
        cfg = self.config
        kv = cfg.n_kv_heads * cfg.head_dim
        d, dff, L = cfg.d_model, cfg.d_ff, cfg.n_layers
        per_layer = (d * (d + 2 * kv) + d * d + 2 * d * dff + dff * d) * 2 + 2 * d * 4
        return L * per_layer + cfg.vocab_size * d * 2 + d * 4


@dataclass
class ModelWeights:
    """Host weights in the reference's file layout (model.py:85-143).  The
    device packing is built once per process on first use (`device()`)."""
    config: ModelConfig
    tensors: dict
    tied_head: bool = True
    _dev: Optional[DeviceModel] = field(default=None, repr=False, compare=False)
    # checkpoint.RopeScaling of an imported HF checkpoint (linear / YaRN /
    # llama3 tables); None = the reference's plain RoPE (tensor.py:66-76)
    rope_scaling: Optional[object] = field(default=None, compare=False)

    def validate(self):
        expected = dict(tensor_order(self.config, self.tied_head))
        if set(expected) != set(self.tensors):
            raise ShapeError(f"weight tensor set mismatch: {sorted(set(expected) ^ set(self.tensors))}")
        for name, shape in expected.items():
            t = self.tensors[name]
            if tuple(t.shape) != shape:
                raise ShapeError(f"{name}: shape {t.shape}, expected {shape}")
            if t.dtype != np.float32:
                raise ShapeError(f"{name}: dtype {t.dtype}, expected float32")
            if not np.isfinite(t).all():
                raise ShapeError(f"{name}: non-finite entries")
        return self

    def checksum(self) -> str:
        h = hashlib.sha256()
        for name, _ in tensor_order(self.config, self.tied_head):
            h.update(name.encode())
            h.update(self.tensors[name].tobytes())
        return h.hexdigest()

    def device(self) -> DeviceModel:
        if self._dev is None:
            self._dev = DeviceModel(self.config, self.tensors, self.tied_head, self.rope_scaling)
        return self._dev

    def runtime(self) -> DeviceModel:
        """Reference name for the packed runtime form (model.py:116)."""
        return self.device()

    def invalidate(self) -> None:
        """Drop the device packing after mutating `tensors` in place (the
        reference's `weights._runtime = None`)."""
        self._dev = None

    def __setattr__(self, name, value):
        if name == "_runtime" and value is None:   # reference idiom: weights._runtime = None
            object.__setattr__(self, "_dev", None)
            return
        object.__setattr__(self, name, value)

    @classmethod
    def on_device(cls, dm: DeviceModel) -> "ModelWeights":
        """Wrap device-only random weights (DeviceModel.random)."""
        w = cls(dm.config, {}, dm.tied_head, rope_scaling=getattr(dm, "rope_scaling", None))
        w._dev = dm
        return w


def generate_weights(config: ModelConfig, seed: int, tied_head: bool = True) -> ModelWeights:
    """Deterministic init, identical stream to the reference (model.py:146-157)."""
    rng = np.random.default_rng(seed)
    tensors = {}
    for name, shape in tensor_order(config, tied_head):
        draw = rng.standard_normal(shape) * 0.02
        tensors[name] = (1.0 + draw if "norm" in name else draw).astype(np.float32)
    return ModelWeights(config, tensors, tied_head).validate()


def plant_successor(weights: ModelWeights, seed: int, easy_frac: float, emb_scale: float = 32.0,
                    margin: float = 24.0) -> ModelWeights:
    """Random-init weights plus a planted next-token channel (benchmark
    workloads; same idea as the reference's planted_attention_weights,
    analytics.py:109-186).

    Independent random-init target and draft models never agree on a greedy
    token, so every speculation is rejected (acceptance 0) and any
    speculative decoder degenerates to several forwards per token.  Real
    long-context pairs accept ~92%.  The plant: a random
    permutation `succ` of the vocabulary and, for a random `easy_frac` subset
    of tokens t, a +-1 direction u_t added to emb[t] (x emb_scale) and to the
    lm_head column of succ(t) (x margin / d_model, so the planted logit
    lead is ~`margin` at any width).  After an easy token every
    model -- whatever its other weights -- puts its argmax on succ(t); after a
    hard token the argmax is decided by the model's own random weights and
    attention, so two different models (or the retrieval and full views of
    one model) disagree.  Acceptance therefore tracks `easy_frac` while every
    forward still runs the full architecture.  Needs an untied head."""
    if weights.tied_head:
        raise ValueError("plant_successor needs an untied lm_head")
    if not 0.0 <= easy_frac <= 1.0:
        raise ValueError("easy_frac must be in [0, 1]")
    cfg = weights.config
    V, d = cfg.vocab_size, cfg.d_model
    rng = np.random.default_rng(seed)
    succ = rng.permutation(V)
    easy = np.nonzero(rng.random(V) < easy_frac)[0]
    u = rng.integers(0, 2, (easy.size, d)).astype(np.float32) * 2.0 - 1.0
    emb = weights.tensors["embedding"]
    head = weights.tensors["lm_head"]
    emb[easy] += np.float32(emb_scale) * u
    head[:, succ[easy]] += np.float32(margin / d) * u.T
    weights.invalidate()
    return weights.validate()


# ---------------------------------------------------------------------------
# tokenizer (model.py:163-176)

def tokenize(data: bytes) -> list:
    return [BOS] + list(data)


def detokenize(tokens: Sequence[int], vocab_size: int = TOKENIZER_VOCAB) -> bytes:
    out = bytearray()
    for t in tokens:
        if not 0 <= t < vocab_size:
            raise ValueError(f"token id {t} outside vocab of size {vocab_size}")
        if t < 256:
            out.append(t)
    return bytes(out)


# ---------------------------------------------------------------------------
# sampling (model.py:182-206) -- device kernels, fp64

def prob_from_logits(logits, temperature: float) -> np.ndarray:
    """fp64 distribution; temperature 0 is a one-hot argmax (lowest index on ties)."""
    if temperature < 0:
        raise ValueError("temperature must be >= 0")
    lg = as_device_f32(logits).reshape(-1)
    out = torch.empty(lg.numel(), dtype=torch.float64, device=lg.device)
    check(lib.hs_probs(ptr(lg), 1, lg.numel(), float(temperature), ptr(out), stream_ptr()))
    return out.cpu().numpy()


def sample_from_probs(probs, rng: np.random.Generator) -> int:
    """Inverse-CDF draw consuming exactly one uniform from `rng`."""
    p = as_device_f64(probs).reshape(-1)
    u = torch.tensor([rng.random()], dtype=torch.float64, device=p.device)
    cur = torch.zeros(1, dtype=torch.int32, device=p.device)
    out = torch.zeros(1, dtype=torch.int32, device=p.device)
    check(lib.hs_sample(ptr(p), p.numel(), ptr(u), ptr(cur), ptr(out), stream_ptr()))
    return int(out.item())


def sample(logits, temperature: float, rng: np.random.Generator) -> int:
    return sample_from_probs(prob_from_logits(logits, temperature), rng)


# ---------------------------------------------------------------------------
# forward passes

@dataclass
class AttentionProbe:
    layer: int
    head: int
    query_position: int
    positions: np.ndarray
    weights: np.ndarray


class ForwardRecorder:
    """Last-row post-RoPE queries of the most recent forward, per layer
    (model.py:222-233).  Kept on the device ([L, H, dh] fp32) so the
    retrieval builder reads it without a host round trip.  record_probs=True
    also records each head's post-softmax attention row of the last query and
    the positions it spans (hs_forward_probe, csrc/h2o.cu) for
    attention_probe and the recovery analytics."""

    def __init__(self, record_probs: bool = False):
        self.record_probs = record_probs
        self.stash: Optional[torch.Tensor] = None
        self.query_position = -1
        self._probs: list = []
        self.positions: list = []

    def _buffer(self, cfg: ModelConfig) -> torch.Tensor:
        shape = (cfg.n_layers, cfg.n_heads, cfg.head_dim)
        if self.stash is None or tuple(self.stash.shape) != shape:
            self.stash = torch.zeros(shape, dtype=torch.float32, device=device())
        return self.stash

    @property
    def last_queries(self) -> list:
        if self.stash is None:
            return []
        host = self.stash.cpu().numpy()
        return [host[i].copy() for i in range(host.shape[0])]

    @property
    def last_probs(self) -> list:
        return self._probs

    def _record(self, cache, step, probe: torch.Tensor) -> None:
        """probe [L][H][n_view] over the view's slots -> per layer the
        visible entries' positions and [H][n] weights (slot order)."""
        host = probe.cpu().numpy()
        n = step.n_view
        qp = step.pos0 + self.query_t - 1
        self._probs, self.positions = [], []
        pos_all = cache.pos[:, :n].cpu().numpy() if cache.pos is not None else None
        for li in range(host.shape[0]):
            kp = pos_all[li] if pos_all is not None else np.arange(n) + step.pos_base
            vis = (kp >= 0) & (kp <= qp)
            if step.window:
                lo = max(qp - step.window + 1, step.win_lo)
                vis &= (kp < step.n_sink) | (kp >= lo)
            self.positions.append(kp[vis].astype(np.int64))
            self._probs.append(host[li][:, vis].astype(np.float32))


PREFILL_MIN_ROWS = 64   # prompts at least this long take the GEMM prefill (hs_prefill)


def forward_device(weights: ModelWeights, tokens, cache, recorder: Optional[ForwardRecorder] = None,
                   out: Optional[torch.Tensor] = None, prefill: bool = False, tp=None) -> torch.Tensor:
    """Causal forward of `tokens` (host list or device int32 tensor) at
    cache.frontier; returns device logits [t, V] fp32 (model.py:247-331).
    prefill=True lets a long prompt on a full cache (unsharded, or
    sequence-sharded at head_dim 128) run through the batched GEMM prefill
    (hs_prefill / hs_prefill_sharded); otherwise every row is computed exactly
    as a decode step would compute it.
    tp: a shard.SequenceShards whose ranks split the dense projections by
    output rows (hs_forward_tp) for blocks of <= 8 rows; longer batches and
    prefill stay replicated."""
    dm = weights.device()
    cfg = dm.config
    tok = to_i32_device(tokens)
    t = tok.numel()
    if t == 0:
        raise ValueError("empty token sequence")
    if not isinstance(tokens, torch.Tensor):
        arr = np.asarray(tokens)
        if arr.min() < 0 or arr.max() >= cfg.vocab_size:
            raise ValueError("token id outside model vocab")
    if cache.frontier + t > cfg.max_seq:
        raise CapacityError(f"sequence of {cache.frontier + t} exceeds max_seq {cfg.max_seq}")
    if out is None:
        out = torch.empty((t, cfg.vocab_size), dtype=torch.float32, device=tok.device)
    stash = recorder._buffer(cfg) if recorder is not None else None
    shards = getattr(cache, "shards", None)
    shard_ref = shards.ref if shards is not None else None
    world = shards.world if shards is not None else 0
    if getattr(cache, "policy", "") == "topk" and t > 1 and not (prefill and cache.frontier == 0):
        # TopKCache selects per single query (caches.py:629-634): a batch is
        # decoded position by position, as the reference's decode_chunk /
        # Lane.advance / token-by-token prefill do (model.py:350-378)
        for i in range(t):
            forward_device(weights, tok[i:i + 1], cache, recorder, out=out[i:i + 1])
        return out
    if recorder is not None and recorder.record_probs:
        return _forward_probe(weights, dm, tok, t, cache, recorder, out, stash, prefill)
    if (prefill and t >= PREFILL_MIN_ROWS and cache.kind == _abi.HS_KV_LINEAR
            and (shards is None or cfg.head_dim == 128)):
        step = cache._step(t)
        if shards is None:
            nbytes = lib.hs_prefill_workspace_bytes(dm.ref, t, step.n_view, step.split)
            ws = workspaces.get("prefill", nbytes)
            check(lib.hs_prefill(dm.ref, cache._ref, C.byref(step), ptr(tok), t, ptr(out), ptr(stash), ptr(ws),
                                 nbytes, stream_ptr()))
        else:   # sequence shards: per-rank partial attention, NCCL exchange, rank-ordered merge
            nbytes = lib.hs_prefill_sharded_workspace_bytes(dm.ref, t, step.n_view, step.split, world)
            ws = workspaces.get("prefill", nbytes)
            check(lib.hs_prefill_sharded(dm.ref, cache._ref, C.byref(step), shard_ref, ptr(tok), t, ptr(out),
                                         ptr(stash), ptr(ws), nbytes, stream_ptr()))
        cache._advance(t)
        if recorder is not None:
            recorder.query_position = cache.frontier - 1
        return out
    if t == 1 and getattr(cache, "policy", "") == "topk" and cache.frontier + 1 > cache.budget:
        step = cache._step(1)                     # TopKCache single-query exposure (caches.py:629-634)
        nbytes = lib.hs_forward_topk_workspace_bytes(dm.ref, step.n_view, cache.budget)
        ws = workspaces.get("topk", nbytes)
        check(lib.hs_forward_topk(dm.ref, cache._ref, C.byref(step), cache.budget, ptr(tok), ptr(out), ptr(stash),
                                  ptr(ws), nbytes, stream_ptr()))
        cache._advance(1)
        if recorder is not None:
            recorder.query_position = cache.frontier - 1
        return out
    if getattr(cache, "wants_attention", False):
        # H2OCache: the forward also reports each query row's head-summed
        # attention probabilities (model.py:306-307), fed to the eviction policy
        for a, b in cache._batches(t):
            step = cache._step(b - a)
            nbytes = lib.hs_forward_workspace_bytes(dm.ref, b - a, step.n_view, step.split, 0)
            ws = dm.workspace(nbytes)
            probs = torch.zeros((cfg.n_layers, b - a, step.n_view), dtype=torch.float64, device=tok.device)
            hp = torch.empty((b - a, cfg.n_heads, step.n_view), dtype=torch.float32, device=tok.device)
            check(lib.hs_forward_attn_probs(dm.ref, cache._ref, C.byref(step), ptr(tok) + 4 * a, b - a,
                                            ptr(out) + 4 * a * cfg.vocab_size, ptr(stash), ptr(probs), ptr(hp),
                                            ptr(ws), nbytes, stream_ptr()))
            pos0 = cache.frontier
            cache._advance(b - a)
            cache.observe_forward(pos0, probs.cpu().numpy())
        if recorder is not None:
            recorder.query_position = cache.frontier - 1
        return out
    for a, b in cache._batches(t):
        step = cache._step(b - a)
        kv_bytes = step.n_view * cfg.n_kv_heads * cfg.head_dim * 4 * cfg.n_layers
        if tp is not None and b - a <= 8:
            nbytes = lib.hs_forward_tp_workspace_bytes(dm.ref, b - a, step.n_view, step.split, world, tp.world)
            ws = dm.workspace(nbytes)
            check(lib.hs_forward_tp(dm.ref, cache._ref, C.byref(step), shard_ref, tp.ref, ptr(tok) + 4 * a, b - a,
                                    ptr(out) + 4 * a * cfg.vocab_size, ptr(stash), ptr(ws), nbytes, stream_ptr()))
            STATS["alg_bytes"] += dm.weight_bytes // tp.world + kv_bytes
        else:
            nbytes = dm.forward_ws_bytes(b - a, step.n_view, step.split, world)
            ws = dm.workspace(nbytes)
            check(lib.hs_forward(dm.ref, cache._ref, C.byref(step), shard_ref, ptr(tok) + 4 * a, b - a,
                                 ptr(out) + 4 * a * cfg.vocab_size, ptr(stash), ptr(ws), nbytes, stream_ptr()))
            STATS["alg_bytes"] += dm.weight_bytes + kv_bytes
        cache._advance(b - a)
    if recorder is not None:
        recorder.query_position = cache.frontier - 1
    return out


def _forward_probe(weights, dm, tok, t, cache, recorder, out, stash, prefill):
    """forward_device with an attention probe of the last row: the rows before
    it take the usual path (GEMM prefill when long), the last one
    hs_forward_probe (model.py:308-312)."""
    if getattr(cache, "shards", None) is not None or getattr(cache, "policy", "") in ("topk", "h2o"):
        raise ContractError("attention probes need an unsharded full, streaming or retrieval cache")
    cfg = dm.config
    if t > 1:
        plain = ForwardRecorder()
        plain.stash = recorder.stash
        forward_device(weights, tok[:t - 1], cache, plain, out=out[:t - 1], prefill=prefill)
    step = cache._step(1)
    nbytes = lib.hs_forward_workspace_bytes(dm.ref, 1, step.n_view, step.split, 0)
    ws = dm.workspace(nbytes)
    probe = torch.zeros((cfg.n_layers, cfg.n_heads, step.n_view), dtype=torch.float32, device=tok.device)
    check(lib.hs_forward_probe(dm.ref, cache._ref, C.byref(step), ptr(tok) + 4 * (t - 1), 1,
                               ptr(out) + 4 * (t - 1) * cfg.vocab_size, ptr(stash), ptr(probe), ptr(ws), nbytes,
                               stream_ptr()))
    recorder.query_t = 1
    recorder._record(cache, step, probe)
    cache._advance(1)
    recorder.query_position = cache.frontier - 1
    return out


def _host_rows(logits: torch.Tensor) -> np.ndarray:
    host = logits.cpu().numpy()
    if not np.isfinite(host).all():
        raise FiniteError("forward produced non-finite logits")
    return host


def prefill(weights: ModelWeights, tokens: Sequence[int], cache,
            recorder: Optional[ForwardRecorder] = None) -> np.ndarray:
    """Append every prompt position, commit, return all logits rows
    (model.py:334-354).  Windowed caches are filled in batches whose
    per-query exposure equals the reference's token-by-token prefill."""
    if len(tokens) == 0:
        raise ValueError("prefill needs at least one token")
    if cache.frontier + len(tokens) > weights.config.max_seq:
        raise CapacityError(f"sequence of {cache.frontier + len(tokens)} exceeds max_seq "
                            f"{weights.config.max_seq}")
    logits = forward_device(weights, tokens, cache, recorder, prefill=True)
    cache.commit(cache.frontier)
    return _host_rows(logits)


def decode_step(weights: ModelWeights, token: int, cache,
                recorder: Optional[ForwardRecorder] = None) -> np.ndarray:
    """One speculative position; next-token logits row (model.py:357-363)."""
    if cache.frontier < 1:
        raise ValueError("decode_step requires a non-empty cache")
    return _host_rows(forward_device(weights, [int(token)], cache, recorder))[0]


def decode_chunk(weights: ModelWeights, tokens: Sequence[int], cache,
                 recorder: Optional[ForwardRecorder] = None) -> np.ndarray:
    """One logits row per token, bit-identical to a decode_step loop
    (model.py:366-378) -- computed as one batched forward."""
    if len(tokens) == 0:
        raise ValueError("empty chunk")
    if cache.frontier < 1:
        raise ValueError("decode_chunk requires a non-empty cache")
    return _host_rows(forward_device(weights, list(tokens), cache, recorder))


def attention_probe(recorder: ForwardRecorder, layer: int, head: int) -> AttentionProbe:
    """One head's attention row from a recorded forward (model.py:381-393)."""
    if not recorder.record_probs or not recorder.last_probs:
        raise ValueError("recorder has no recorded attention (pass record_probs=True)")
    if not 0 <= layer < len(recorder.last_probs):
        raise IndexError(f"layer {layer} out of range")
    row = recorder.last_probs[layer]
    if not 0 <= head < row.shape[0]:
        raise IndexError(f"head {head} out of range")
    return AttentionProbe(layer=layer, head=head, query_position=recorder.query_position,
                          positions=recorder.positions[layer], weights=row[head])
