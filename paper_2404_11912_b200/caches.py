"""KV-cache policies on the device -- the drop-in for hierspec/caches.py.

Bookkeeping contract (caches.py:1-19): `frontier` is the next position to
append, positions >= `committed` are speculative, `rollback_to(n)` drops
positions >= n, `commit(n)` promotes positions < n and applies the policy's
eviction/overwrite rule.

Device layout: K and V are bf16 [layer][kv_head][slot][head_dim]
(head-major, so one head's keys stream contiguously); slotted caches keep
an int32 absolute position per (layer, slot).

* FullCache        slot == position.
* StreamingCache   sinks at slots [0, n_sink), the recent window in a ring
                   slot = n_sink + (p - n_sink) % ring; eviction is a host
                   watermark (`lo`) -- nothing moves on the device.
* RetrievalCache   selected chunks in slots [0, n_sel) (position order after
                   a build), speculative tail in [n_sel, n_sel + n_spec);
                   the victim FIFO is a fixed ring of slot indices.

The per-layer `append`/`expose` hooks of the reference protocol are kept for
API compatibility and tests; the fused forward (`hs_forward`) writes and
reads the caches directly and never materialises `expose()`.
"""

from __future__ import annotations

import os

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from ._abi import (HS_APPEND_LINEAR, HS_APPEND_POS, HS_APPEND_RING, HS_KV_LINEAR, HS_KV_SLOTTED, HsCache,
                   HsStep, check, lib)
from .errors import CapacityError, ContractError, ShapeError
from .runtime import STATS, as_device_f32, device, ptr, stream_ptr

FULL_SPLIT = int(os.environ.get("HS_FULL_SPLIT", 2048))    # keys per attention split over the full cache
SMALL_SPLIT = int(os.environ.get("HS_SMALL_SPLIT", 512))   # keys per split over the retrieval view
# (fixed per cache kind, never a function of t: a row's result is t-invariant;
# the environment overrides are experiment hooks for tools/fwdbench.py)
STREAM_SPLIT = int(os.environ.get("HS_STREAM_SPLIT", 64))   # keys per split over the streaming window


def stream_split(head_dim: int) -> int:
    """Split for streaming / H2O views: the tensor-core kernel (head_dim 128)
    walks 128-key tiles, so its splits are whole tiles."""
    return STREAM_SPLIT if head_dim < 128 else max(128, STREAM_SPLIT // 128 * 128)


@dataclass(frozen=True)
class StreamingConfig:
    """caches.py:32-39"""
    n_sink: int = 4
    budget: int = 64

    def __post_init__(self):
        if not 0 <= self.n_sink < self.budget:
            raise ValueError("need 0 <= n_sink < budget")


@dataclass(frozen=True)
class H2OConfig:
    """caches.py:42-49 (H2OCache below)."""
    budget: int = 64
    recent_window: int = 32

    def __post_init__(self):
        if not 0 <= self.recent_window < self.budget:
            raise ValueError("need 0 <= recent_window < budget")


@dataclass(frozen=True)
class RetrievalConfig:
    """caches.py:52-68"""
    chunk_size: int = 16
    budget: int = 64
    rebuild_stride: int = 128
    rebuild_accept_threshold: float = 0.8
    rolling_window: int = 16

    def __post_init__(self):
        if self.chunk_size < 1 or self.budget < self.chunk_size:
            raise ValueError("need chunk_size >= 1 and budget >= chunk_size")
        if self.budget % self.chunk_size:
            raise ValueError("budget must be a multiple of chunk_size")
        if not 0.0 < self.rebuild_accept_threshold < 1.0:
            raise ValueError("rebuild_accept_threshold must be in (0, 1)")
        if self.rebuild_stride < 1 or self.rolling_window < 1:
            raise ValueError("rebuild_stride and rolling_window must be >= 1")


class KVCache:
    """Base: device buffers, descriptor, bookkeeping helpers."""

    policy = "base"
    wants_attention = False
    batched_prefill_ok = True
    kind = HS_KV_LINEAR

    def __init__(self, n_layers: int, n_kv_heads: int, head_dim: int, cap: int, with_pos: bool):
        self.n_layers, self.n_kv_heads, self.head_dim = n_layers, n_kv_heads, head_dim
        self.frontier = 0
        self.committed = 0
        self.cap = cap
        dev = device()
        self.k = torch.zeros((n_layers, n_kv_heads, cap, head_dim), dtype=torch.bfloat16, device=dev)
        self.v = torch.zeros_like(self.k)
        self.pos = torch.full((n_layers, cap), -1, dtype=torch.int32, device=dev) if with_pos else None
        d = HsCache()
        d.kind, d.n_layers, d.n_kv_heads, d.head_dim, d.cap = self.kind, n_layers, n_kv_heads, head_dim, cap
        d.k, d.v, d.pos = self.k.data_ptr(), self.v.data_ptr(), ptr(self.pos)
        self._desc = d
        self._ref = C.byref(d)

    @classmethod
    def from_config(cls, model_config, *args, **kwargs):
        return cls(model_config.n_layers, model_config.n_kv_heads, model_config.head_dim, *args, **kwargs)

    # -- protocol ----------------------------------------------------------------
    def observe_attention(self, layer, probs, query_positions):
        pass

    def _check_kv(self, k, v):
        if tuple(k.shape) != tuple(v.shape) or k.ndim != 3 or tuple(k.shape[1:]) != (self.n_kv_heads, self.head_dim):
            raise ShapeError(f"bad kv shape {tuple(k.shape)}")

    def _check_commit(self, n: int):
        if not self.committed <= n <= self.frontier:
            raise ContractError(f"commit({n}) outside [{self.committed}, {self.frontier}]")

    def _write_rows(self, layer: int, k, v, slots, positions):
        kd, vd = as_device_f32(k), as_device_f32(v)
        s = torch.as_tensor(np.asarray(slots, np.int32)).to(kd.device)
        p = torch.as_tensor(np.asarray(positions, np.int32)).to(kd.device)
        check(lib.hs_kv_write(self._ref, layer, ptr(kd), ptr(vd), kd.shape[0], ptr(s), ptr(p), stream_ptr()))

    def _gather_host(self, layer: int, slots: np.ndarray):
        idx = torch.as_tensor(np.asarray(slots, np.int64), device=self.k.device)
        K = self.k[layer].index_select(1, idx).permute(1, 0, 2).float().cpu().numpy()
        V = self.v[layer].index_select(1, idx).permute(1, 0, 2).float().cpu().numpy()
        return K, V

    def exposed_positions(self, layer: int = 0) -> np.ndarray:
        return np.asarray(self.expose(layer)[2]).copy()

    def to_json(self) -> dict:
        return {"policy": self.policy, "frontier": self.frontier, "committed": self.committed,
                "layers": [{"exposed_positions": np.asarray(self.expose(li)[2]).tolist()}
                           for li in range(self.n_layers)]}

    # -- fused-forward hooks (overridden) ------------------------------------------
    def _batches(self, t: int):
        yield 0, t

    def _step(self, t: int) -> HsStep:
        raise NotImplementedError

    def _advance(self, t: int) -> None:
        raise NotImplementedError


class FullCache(KVCache):
    """Keeps every position (caches.py:176-221); capacity = max_entries.

    Sequence-sharded form (`FullCache.shard`): this rank
    stores positions [lo, hi) (hi None = the tail, up to max_entries) in
    slots 0.. ; frontier / committed stay global and every forward merges
    the per-rank attention states over NCCL (shard.py)."""

    policy = "full"
    kind = HS_KV_LINEAR

    def __init__(self, n_layers: int, n_kv_heads: int, head_dim: int, max_entries: int,
                 shards=None, lo: int = 0, hi: Optional[int] = None):
        if lo < 0 or (hi is not None and not lo < hi <= max_entries) or lo >= max_entries:
            raise ValueError(f"bad shard range [{lo}, {hi}) for max_entries {max_entries}")
        local = (hi if hi is not None else max_entries) - lo
        super().__init__(n_layers, n_kv_heads, head_dim, local, with_pos=False)
        self.max_entries = max_entries
        self.shards, self.lo, self.hi = shards, lo, hi
        self.bounds = [(lo, hi)]
        self._n = [0] * n_layers

    @classmethod
    def from_config(cls, model_config):
        return cls(model_config.n_layers, model_config.n_kv_heads, model_config.head_dim, model_config.max_seq)

    @classmethod
    def shard(cls, model_config, shards, n_context: int, chunk: int):
        """This rank's shard of a full cache whose first n_context positions
        are split by shard.shard_plan (chunk-aligned)."""
        plan = shards.plan(n_context, chunk)
        lo, hi = plan[shards.rank]
        c = cls(model_config.n_layers, model_config.n_kv_heads, model_config.head_dim, model_config.max_seq,
                shards, lo, hi)
        c.bounds = plan
        return c

    @property
    def sharded(self) -> bool:
        return self.shards is not None

    def _local(self, n: int) -> int:
        """slots of this rank holding positions < n"""
        return max(0, min(n - self.lo, self.cap))

    def append(self, layer, k, v):
        self._check_kv(k, v)
        t = k.shape[0]
        n = self._n[layer]
        if n + t > self.max_entries:
            raise CapacityError(f"full cache overflow past {self.max_entries}")
        pos = np.arange(n, n + t)
        keep = (pos >= self.lo) & (pos < self.lo + self.cap)
        if keep.any():
            kd, vd = as_device_f32(k), as_device_f32(v)
            idx = torch.as_tensor(np.nonzero(keep)[0], device=kd.device)
            self._write_rows(layer, kd.index_select(0, idx), vd.index_select(0, idx), pos[keep] - self.lo, pos[keep])
        self._n[layer] = n + t
        if layer == self.n_layers - 1:
            self.frontier = n + t

    def expose(self, layer, queries=None):
        """This rank's positions (all of them when unsharded)."""
        m = self._local(self._n[layer])
        K, V = self._gather_host(layer, np.arange(m))
        return K, V, np.arange(self.lo, self.lo + m, dtype=np.int64), None

    def rollback_to(self, n):
        self._n = [min(x, n) for x in self._n]
        self.frontier = min(self.frontier, n)
        self.committed = min(self.committed, n)

    def commit(self, n):
        self._check_commit(n)
        self.committed = n

    def clone(self):
        c = FullCache(self.n_layers, self.n_kv_heads, self.head_dim, self.max_entries, self.shards, self.lo, self.hi)
        c.bounds = list(self.bounds)
        check(lib.hs_cache_copy(c._ref, self._ref, self._local(max(self._n + [0])), stream_ptr()))
        c._n = list(self._n)
        c.frontier, c.committed = self.frontier, self.committed
        return c

    def fill_random_(self, n: int, seed: int = 0, std: float = 1.0):
        """Synthetic context: n committed positions of N(0, std) bf16 K/V
        (throughput configs).  Each shard fills its own
        positions from a stream keyed by (seed, lo)."""
        if n > self.max_entries:
            raise CapacityError("fill beyond capacity")
        g = torch.Generator(device=self.k.device)
        g.manual_seed(seed * 1000003 + self.lo)
        m = self._local(n)
        for l in range(self.n_layers):
            for h in range(self.n_kv_heads):
                self.k[l, h, :m].normal_(0.0, std, generator=g)
                self.v[l, h, :m].normal_(0.0, std, generator=g)
        self._n = [n] * self.n_layers
        self.frontier = self.committed = n

    # fused forward: append at slot == position - lo, attend to this rank's slots
    def _step(self, t):
        s = HsStep()
        s.pos0 = self.frontier
        s.append_mode = HS_APPEND_POS
        if self.frontier + t > self.max_entries:
            raise CapacityError(f"full cache overflow past {self.max_entries}")
        s.n_view = self._local(self.frontier + t)
        s.split = FULL_SPLIT
        s.pos_base = self.lo
        s.own_hi = self.hi if self.hi is not None else 0
        return s

    def _advance(self, t):
        self.frontier += t
        self._n = [self.frontier] * self.n_layers


class H2OCache(KVCache):
    """Heavy-hitter eviction (caches.py:291-396): per layer, cumulative
    attention probabilities summed across heads; at commit the lowest-score
    committed entry outside the recent window is evicted (ties to the oldest
    position) until the committed set fits the budget.  Scores earned by
    speculative queries stay pending until the query's position commits.

    Device layout: a slotted cache with slot == position (entries are never
    moved; an evicted entry's position becomes -1, so the attention kernels
    skip it).  The probabilities come from hs_forward_attn_probs (csrc/h2o.cu)
    with the reference's rounding points; the pending / score / eviction
    bookkeeping is host logic over them, as in the reference."""

    policy = "h2o"
    wants_attention = True
    kind = HS_KV_SLOTTED

    def __init__(self, n_layers: int, n_kv_heads: int, head_dim: int, config: H2OConfig, max_entries: int = 4096):
        super().__init__(n_layers, n_kv_heads, head_dim, max_entries, with_pos=True)
        self.config = config
        self.max_entries = max_entries
        self._alive = np.zeros((n_layers, max_entries), dtype=bool)
        self._scores = np.zeros((n_layers, max_entries), dtype=np.float64)
        self._pending = [[] for _ in range(n_layers)]
        self._nl = [0] * n_layers   # entries appended per layer (slot == position)

    @classmethod
    def from_config(cls, model_config, config: H2OConfig):
        return cls(model_config.n_layers, model_config.n_kv_heads, model_config.head_dim, config,
                   model_config.max_seq)

    def _step(self, t):
        if self.frontier + t > self.max_entries:
            raise CapacityError(f"h2o cache overflow past {self.max_entries}")
        s = HsStep()
        s.pos0 = self.frontier
        s.append_mode = HS_APPEND_LINEAR
        s.append_base = self.frontier
        s.n_view = self.frontier + t
        s.split = stream_split(self.head_dim)
        return s

    def _advance(self, t):
        a, b = self.frontier, self.frontier + t
        self._alive[:, a:b] = True
        self._scores[:, a:b] = 0.0
        self.frontier = b
        self._nl = [b] * self.n_layers

    # -- per-layer protocol (KVCache.append / observe_attention, caches.py:311-345) --
    def append(self, layer, k, v):
        self._check_kv(k, v)
        t = k.shape[0]
        n = self._nl[layer]
        if n + t > self.max_entries:
            raise CapacityError(f"h2o cache overflow past {self.max_entries}")
        pos = np.arange(n, n + t)
        self._write_rows(layer, k, v, pos, pos)
        self._alive[layer, n:n + t] = True
        self._scores[layer, n:n + t] = 0.0
        self._nl[layer] = n + t
        if layer == self.n_layers - 1:
            self.frontier = n + t

    def observe_attention(self, layer, probs, query_positions):
        """probs [KVH, g, t, L] over this layer's exposed entries (position order)."""
        slots = np.nonzero(self._alive[layer, :self._nl[layer]])[0]
        p = np.asarray(probs)
        if p.shape[-1] != slots.size:
            raise ShapeError(f"attention row spans {p.shape[-1]} entries, layer exposes {slots.size}")
        rows = p.astype(np.float64).sum(axis=(0, 1))
        for i, qpos in enumerate(np.asarray(query_positions)):
            self._pending[layer].append((int(qpos), slots, rows[i].copy()))

    def observe_forward(self, pos0: int, probs: np.ndarray) -> None:
        """probs [L][t][n_view]: each new query row's head-summed attention
        probabilities over the exposed slots (H2OCache.observe_attention)."""
        t = probs.shape[1]
        for li in range(self.n_layers):
            slots = np.nonzero(self._alive[li, :probs.shape[2]])[0]
            for i in range(t):
                self._pending[li].append((pos0 + i, slots, probs[li, i, slots].copy()))

    def expose(self, layer, queries=None):
        slots = np.nonzero(self._alive[layer, :self._nl[layer]])[0]
        K, V = self._gather_host(layer, slots)
        return K, V, slots.astype(np.int64), None

    def rollback_to(self, n):
        if n < self.committed:
            raise ContractError(f"h2o cache cannot roll below committed {self.committed}")
        if n < self.frontier:
            self._alive[:, n:self.frontier] = False
            self.pos[:, n:self.frontier] = -1
        for li in range(self.n_layers):
            self._pending[li] = [p for p in self._pending[li] if p[0] < n]
        self.frontier = min(self.frontier, n)
        self._nl = [min(x, n) for x in self._nl]

    def commit(self, n):
        self._check_commit(n)
        self.committed = n
        cfg = self.config
        dead = []
        for li in range(self.n_layers):
            alive, scores = self._alive[li], self._scores[li]
            keep = []
            for qpos, slots, w in self._pending[li]:
                if qpos >= n:
                    keep.append((qpos, slots, w))
                    continue
                ok = alive[slots]
                scores[slots[ok]] += w[ok]
            self._pending[li] = keep
            while True:   # caches.py:374-388
                pos = np.nonzero(alive[:self.frontier])[0]
                comm = pos[pos < n]
                if comm.size <= cfg.budget:
                    break
                recent_cut = comm[-cfg.recent_window] if cfg.recent_window else n
                cand = comm[comm < recent_cut]
                victim = cand[np.lexsort((cand, scores[cand]))[0]]
                alive[victim] = False
                dead.append((li, victim))
        if dead:
            idx = torch.as_tensor(np.asarray(dead, dtype=np.int64).T, device=self.pos.device)
            self.pos[idx[0], idx[1]] = -1

    def cumulative_scores(self, layer: int) -> dict:
        slots = np.nonzero(self._alive[layer, :self.frontier])[0]
        return {int(p): float(self._scores[layer, p]) for p in slots}

    def clone(self):
        c = H2OCache(self.n_layers, self.n_kv_heads, self.head_dim, self.config, self.max_entries)
        check(lib.hs_cache_copy(c._ref, self._ref, self.frontier, stream_ptr()))
        c._alive = self._alive.copy()
        c._scores = self._scores.copy()
        c._pending = [[(q, s.copy(), w.copy()) for q, s, w in pl] for pl in self._pending]
        c._nl = list(self._nl)
        c.frontier, c.committed = self.frontier, self.committed
        return c


class TopKCache(FullCache):
    """Oracle upper bound (caches.py:568-652): keeps every position like the
    full cache and, for each single-query decode, each layer attends only
    over the `budget` entries per kv group with the highest exact group-mean
    softmax weight (ties to the lower position); multi-query forwards, and
    stores of at most `budget` entries, see everything.  The selection runs on
    the device inside hs_forward_topk (csrc/topk.cu)."""

    policy = "topk"

    def __init__(self, n_layers: int, n_kv_heads: int, head_dim: int, max_entries: int, budget: int):
        if budget < 1:
            raise ValueError("budget must be >= 1")
        super().__init__(n_layers, n_kv_heads, head_dim, max_entries)
        self.budget = budget

    @classmethod
    def from_config(cls, model_config, budget: int):
        return cls(model_config.n_layers, model_config.n_kv_heads, model_config.head_dim, model_config.max_seq,
                   budget)

    def clone(self):
        c = TopKCache(self.n_layers, self.n_kv_heads, self.head_dim, self.max_entries, self.budget)
        check(lib.hs_cache_copy(c._ref, self._ref, max(self._n + [0]), stream_ptr()))
        c._n = list(self._n)
        c.frontier, c.committed = self.frontier, self.committed
        return c


class StreamingCache(KVCache):
    """Attention sinks + recent window (caches.py:224-288).

    Store = positions [0, n_sink) U [lo, hi); exposure for a query at p is
    the sinks plus [max(lo, p - W + 1), p] with W = budget - n_sink -- the
    reference's `expose` evaluated after appending p.  Commit raises the
    watermark lo to max(lo, n - W) (keep the last W committed)."""

    policy = "streaming"
    batched_prefill_ok = False
    kind = HS_KV_SLOTTED

    def __init__(self, n_layers: int, n_kv_heads: int, head_dim: int, config: StreamingConfig,
                 slack: int = 128):
        self.config = config
        self.window = config.budget - config.n_sink
        self.ring = self.window + slack
        self.slack = slack
        super().__init__(n_layers, n_kv_heads, head_dim, config.n_sink + self.ring, with_pos=True)
        self.lo = config.n_sink
        self._hi = [0] * n_layers

    def _slot(self, p: int) -> int:
        ns = self.config.n_sink
        return p if p < ns else ns + (p - ns) % self.ring

    def _store(self, hi: int) -> np.ndarray:
        ns = self.config.n_sink
        return np.concatenate([np.arange(min(ns, hi)), np.arange(max(self.lo, ns), hi)]).astype(np.int64)

    def _guard(self, first_new: int, last_new: int):
        """Appending up to last_new overwrites last_new - ring; that position
        must no longer be exposable (current or after a rollback to committed)."""
        base = self.committed if self.committed > 0 else first_new
        lowest = max(self.lo, base - self.window + 1)
        if last_new - self.ring >= lowest:
            raise CapacityError(f"streaming ring ({self.ring} slots) too small for the speculative tail; "
                                f"raise slack")

    def append(self, layer, k, v):
        self._check_kv(k, v)
        t = k.shape[0]
        p0 = self.frontier
        self._guard(p0, p0 + t - 1)
        pos = np.arange(p0, p0 + t)
        self._write_rows(layer, k, v, [self._slot(int(p)) for p in pos], pos)
        self._hi[layer] = p0 + t
        if layer == self.n_layers - 1:
            self.frontier = p0 + t

    def _exposed(self, hi: int) -> np.ndarray:
        st = self._store(hi)
        if st.shape[0] <= self.config.budget:
            return st
        return np.concatenate([st[:self.config.n_sink], st[-self.window:]])

    def expose(self, layer, queries=None):
        pos = self._exposed(self._hi[layer])
        K, V = self._gather_host(layer, [self._slot(int(p)) for p in pos])
        return K, V, pos, None

    def rollback_to(self, n):
        if n < self.committed:
            raise ContractError(f"streaming cache cannot roll below committed {self.committed}")
        self._hi = [min(h, n) for h in self._hi]
        self.frontier = min(self.frontier, n)

    def commit(self, n):
        self._check_commit(n)
        self.committed = n
        ns = self.config.n_sink
        n_comm = min(n, ns) + max(0, n - max(self.lo, ns))
        if n_comm > self.config.budget:
            self.lo = max(self.lo, n - self.window)

    def clone(self):
        c = StreamingCache(self.n_layers, self.n_kv_heads, self.head_dim, self.config, self.slack)
        check(lib.hs_cache_copy(c._ref, self._ref, self.cap, stream_ptr()))
        c._hi, c.lo = list(self._hi), self.lo
        c.frontier, c.committed = self.frontier, self.committed
        return c

    def fill_random_(self, n: int, seed: int = 0, std: float = 1.0):
        """Synthetic state equal to 'prefilled n positions and committed'."""
        ns = self.config.n_sink
        g = torch.Generator(device=self.k.device)
        g.manual_seed(seed)
        self.lo = ns
        self.frontier = n
        self._hi = [n] * self.n_layers
        keep = self._store(n)
        if keep.shape[0] > self.config.budget:
            self.lo = n - self.window
            keep = self._store(n)
        slots = torch.as_tensor([self._slot(int(p)) for p in keep], device=self.k.device)
        for l in range(self.n_layers):
            kk = torch.randn((self.n_kv_heads, len(keep), self.head_dim), generator=g, device=self.k.device) * std
            vv = torch.randn((self.n_kv_heads, len(keep), self.head_dim), generator=g, device=self.k.device) * std
            self.k[l][:, slots] = kk.to(torch.bfloat16)
            self.v[l][:, slots] = vv.to(torch.bfloat16)
            self.pos[l, slots] = torch.as_tensor(keep, dtype=torch.int32, device=self.k.device)
        self.committed = n

    # fused forward
    def _batches(self, t):
        step = max(1, self.slack // 2)
        for a in range(0, t, step):
            yield a, min(t, a + step)

    def _step(self, t):
        self._guard(self.frontier, self.frontier + t - 1)
        s = HsStep()
        s.pos0 = self.frontier
        s.append_mode = HS_APPEND_RING
        s.n_sink = self.config.n_sink
        s.ring = self.ring
        s.n_view = self.cap
        s.window = self.window
        s.win_lo = self.lo
        s.split = stream_split(self.head_dim)
        return s

    def _advance(self, t):
        self.frontier += t
        self._hi = [self.frontier] * self.n_layers


class ChunkScoreTable:
    """Per-layer chunk-scoring snapshot of a build (caches.py:399-411).
    Device results are copied to the host on first access."""

    def __init__(self, chunk_size, upto, n_layers, scores_dev, importance_dev, n_imp, clamped):
        self.chunk_size = chunk_size
        self.clamped = clamped
        n = (upto + chunk_size - 1) // chunk_size
        b = np.minimum(np.arange(n + 1) * chunk_size, upto).astype(np.int64)
        self.boundaries = [b.copy() for _ in range(n_layers)]
        self._scores_dev, self._imp_dev, self._n_imp = scores_dev, importance_dev, n_imp
        self._scores = self._selected = None

    @property
    def scores(self):
        if self._scores is None:
            h = self._scores_dev.cpu().numpy()
            self._scores = [h[i].copy() for i in range(h.shape[0])]
        return self._scores

    @property
    def selected(self):
        if self._selected is None:
            h = self._imp_dev.cpu().numpy()
            self._selected = [h[i, :self._n_imp].astype(int).tolist() for i in range(h.shape[0])]
        return self._selected

    def ranking(self, layer: int) -> list:
        s = self.scores[layer]
        return sorted(range(len(s)), key=lambda c: (-s[c], c))


def _queries_device(queries, n_layers: int) -> torch.Tensor:
    if isinstance(queries, torch.Tensor):
        q = queries.to(device=device(), dtype=torch.float32)
    else:
        q = torch.from_numpy(np.stack([np.asarray(x, np.float32) for x in queries])).to(device())
    if q.dim() != 3 or q.shape[0] != n_layers:
        raise ShapeError(f"queries must be [n_layers, n_heads, head_dim], got {tuple(q.shape)}")
    return q.contiguous()


def score_chunks(keys, queries, chunk_size: int, n_kv_heads: int):
    """Chunk scores for one layer (caches.py:414-436): mean over query heads
    of q_h . mean_key[h // g] / sqrt(dh), fp64, on the device.
    keys [L, KVH, dh] fp32, queries [H, dh]; returns (bounds, scores)."""
    k = as_device_f32(keys)
    q = as_device_f32(queries)
    if k.dim() != 3 or q.dim() != 2 or k.shape[2] != q.shape[1] or k.shape[1] != n_kv_heads:
        raise ShapeError("score_chunks: keys [L, KVH, dh], queries [H, dh]")
    L, KVH, dh = k.shape
    n = (L + chunk_size - 1) // chunk_size
    out = torch.empty((1, n), dtype=torch.float64, device=k.device)
    check(lib.hs_chunk_score(ptr(k), 0, 0, dh, KVH * dh, 1, KVH, dh, L, chunk_size, ptr(q), q.shape[0],
                             ptr(out), stream_ptr()))
    bounds = np.minimum(np.arange(n + 1) * chunk_size, L).astype(np.int64)
    return bounds, out[0].cpu().numpy()


class RetrievalCache(KVCache):
    """Budgeted chunk-selected view of a full cache (caches.py:439-565)."""

    policy = "retrieval"
    batched_prefill_ok = False
    kind = HS_KV_SLOTTED

    def __init__(self, n_layers: int, n_kv_heads: int, head_dim: int, config: RetrievalConfig,
                 spec_cap: int = 64):
        self.config = config
        self.spec_cap = spec_cap
        super().__init__(n_layers, n_kv_heads, head_dim, config.budget + spec_cap, with_pos=True)
        dev = device()
        self.quota = config.budget // config.chunk_size
        self.ring = torch.zeros((n_layers, config.budget), dtype=torch.int32, device=dev)
        self.importance = torch.zeros((n_layers, self.quota), dtype=torch.int32, device=dev)
        self.chosen = torch.zeros((n_layers, self.quota), dtype=torch.int32, device=dev)
        self.counts = torch.zeros(2, dtype=torch.int32, device=dev)
        self.n_sel = 0
        self.ring_head = 0
        self.n_spec = [0] * n_layers
        self.table: Optional[ChunkScoreTable] = None
        self.builds = 0

    def build(self, source: FullCache, queries, upto: int) -> ChunkScoreTable:
        """Select chunks of source positions [0, upto) with per-layer queries
        [H, dh]; replaces the selection and the speculative tail; frontier =
        committed = upto (caches.py:458-502).  Runs entirely on the device."""
        if upto < 1:
            raise ContractError("retrieval build needs a non-empty source prefix")
        if min(source._n) < upto:
            raise ContractError("source cache shorter than requested build range")
        cfg = self.config
        q = _queries_device(queries, self.n_layers)
        n = (upto + cfg.chunk_size - 1) // cfg.chunk_size
        scores = self._score(source, q, upto, n)
        check(lib.hs_chunk_select(ptr(scores), self.n_layers, n, upto, cfg.chunk_size, cfg.budget,
                                  ptr(self.importance), ptr(self.chosen), ptr(self.ring), ptr(self.counts),
                                  None, 0, stream_ptr()))
        clamped = cfg.budget >= upto
        k_sel = min(n - 1, self.quota - 1)
        n_chosen = k_sel + 1
        self.n_sel = k_sel * cfg.chunk_size + (upto - (n - 1) * cfg.chunk_size)
        self.pos.fill_(-1)
        check(lib.hs_retrieval_gather(source._ref, self._ref, ptr(self.chosen), self.quota, n_chosen,
                                      cfg.chunk_size, upto, source.lo, source.hi or 0, stream_ptr()))
        if source.sharded:
            self._exchange(source, n_chosen, upto)
        self.ring_head = 0
        self.n_spec = [0] * self.n_layers
        self.frontier = self.committed = upto
        self.builds += 1
        row = self.n_kv_heads * self.head_dim * 2 * self.n_layers
        STATS["alg_bytes"] += source._local(upto) * row + self.n_sel * row * 4   # K read + K,V gather r/w
        self.table = ChunkScoreTable(cfg.chunk_size, upto, self.n_layers, scores, self.importance, n_chosen,
                                     clamped)
        return self.table

    def _exchange(self, source: FullCache, n_chosen: int, upto: int) -> None:
        """Sharded build: every rank has gathered the chosen chunks it stores
        (chunks never straddle shards, and the chosen list is ascending, so
        each rank's chunks are one contiguous slot range per layer).  The
        ranges are exchanged so every rank holds the whole selection -- each
        byte crosses the fabric once (hs_retrieval_exchange)."""
        cfg, sh = self.config, source.shards
        ch = self.chosen[:, :n_chosen].cpu().numpy().astype(np.int64)      # replicated selection
        los = np.array([lo for lo, _ in source.bounds], dtype=np.int64)
        owner = np.searchsorted(los, ch * cfg.chunk_size, side="right") - 1  # [L, n_chosen]
        ranges = np.zeros((self.n_layers, sh.world, 2), dtype=np.int32)
        for l in range(self.n_layers):
            first = np.searchsorted(owner[l], np.arange(sh.world), side="left")
            last = np.searchsorted(owner[l], np.arange(sh.world), side="right")
            ranges[l, :, 0] = np.minimum(first * cfg.chunk_size, self.n_sel)
            ranges[l, :, 1] = np.minimum(last * cfg.chunk_size, self.n_sel)
        nb = lib.hs_retrieval_exchange_workspace_bytes(self._ref)
        from .runtime import workspaces
        ws = workspaces.get("retrieval_exchange", nb)
        check(lib.hs_retrieval_exchange(sh.ref, self._ref, ranges.ctypes.data, ptr(ws), nb, stream_ptr()))

    def _score(self, source: FullCache, q: torch.Tensor, upto: int, n: int) -> torch.Tensor:
        """fp64 chunk scores [L, n] of source positions [0, upto).  Sharded:
        each rank scores the chunks it stores (chunk-aligned shards), the
        per-rank rows are all-gathered and concatenated in rank order --
        bit-identical to the unsharded scores (chunks are independent)."""
        cfg, dh = self.config, self.head_dim
        dev = q.device

        def local_scores(count, local_upto):
            out = torch.empty((self.n_layers, count), dtype=torch.float64, device=dev)
            if count:
                check(lib.hs_chunk_score(ptr(source.k), 1, self.n_kv_heads * source.cap * dh, source.cap * dh, dh,
                                         self.n_layers, self.n_kv_heads, dh, local_upto, cfg.chunk_size, ptr(q),
                                         q.shape[1], ptr(out), stream_ptr()))
            return out

        if not source.sharded:
            return local_scores(n, upto)
        from .shard import shard_chunk_counts
        sh = source.shards
        if any(lo % cfg.chunk_size for lo, _ in source.bounds):
            raise ContractError("shard boundaries must be multiples of the retrieval chunk size")
        counts = shard_chunk_counts(source.bounds, upto, cfg.chunk_size)
        cmax = max(counts)
        mine = counts[sh.rank]
        send = torch.zeros((self.n_layers, cmax), dtype=torch.float64, device=dev)
        if mine:
            send[:, :mine] = local_scores(mine, min(upto, source.lo + source.cap) - source.lo)
        recv = sh.all_gather(send)
        scores = torch.cat([recv[r, :, :counts[r]] for r in range(sh.world)], dim=1).contiguous()
        if scores.shape[1] != n:
            raise ContractError(f"sharded scores cover {scores.shape[1]} chunks, expected {n}")
        return scores

    def append(self, layer, k, v):
        self._check_kv(k, v)
        t = k.shape[0]
        ns = self.n_spec[layer]
        if ns + t > self.spec_cap:
            raise CapacityError("retrieval speculative tail overflow")
        p0 = self.frontier
        self._write_rows(layer, k, v, np.arange(self.n_sel + ns, self.n_sel + ns + t), np.arange(p0, p0 + t))
        self.n_spec[layer] = ns + t
        if layer == self.n_layers - 1:
            self.frontier = p0 + t

    def expose(self, layer, queries=None):
        pos_all = self.pos[layer, :self.n_sel + self.n_spec[layer]].cpu().numpy().astype(np.int64)
        sel = pos_all[:self.n_sel]
        order = np.argsort(sel, kind="stable")     # reference keeps sel position-sorted
        slots = np.concatenate([order, np.arange(self.n_sel, self.n_sel + self.n_spec[layer])])
        K, V = self._gather_host(layer, slots)
        return K, V, pos_all[slots], None

    def rollback_to(self, n):
        if n < self.committed:
            raise ContractError(f"retrieval cache cannot roll below committed {self.committed}")
        self.n_spec = [max(0, min(s, n - self.committed)) for s in self.n_spec]
        self.frontier = min(self.frontier, n)

    def commit(self, n):
        self._check_commit(n)
        take = n - self.committed
        if take > 0:
            if self.n_sel < 1:
                raise ContractError("retrieval cache has no slots")
            spec = self.n_spec[0]
            check(lib.hs_retrieval_commit(self._ref, ptr(self.ring), self.config.budget, self.n_sel, self.ring_head, spec, take,
                                          stream_ptr()))
            self.ring_head = (self.ring_head + take) % self.n_sel
            self.n_spec = [s - take for s in self.n_spec]
        self.committed = n

    def clone(self):
        c = RetrievalCache(self.n_layers, self.n_kv_heads, self.head_dim, self.config, self.spec_cap)
        check(lib.hs_cache_copy(c._ref, self._ref, self.cap, stream_ptr()))
        c.ring.copy_(self.ring)
        c.importance.copy_(self.importance)
        c.chosen.copy_(self.chosen)
        c.n_sel, c.ring_head, c.n_spec = self.n_sel, self.ring_head, list(self.n_spec)
        c.frontier, c.committed, c.table, c.builds = self.frontier, self.committed, self.table, self.builds
        return c

    # fused forward: tail appended linearly after the selection
    def _batches(self, t):
        step = self.spec_cap
        for a in range(0, t, step):
            yield a, min(t, a + step)

    def _step(self, t):
        ns = self.n_spec[0]
        if ns + t > self.spec_cap:
            raise CapacityError("retrieval speculative tail overflow")
        s = HsStep()
        s.pos0 = self.frontier
        s.append_mode = HS_APPEND_LINEAR
        s.append_base = self.n_sel + ns
        s.n_view = self.n_sel + ns + t
        s.split = SMALL_SPLIT
        return s

    def _advance(self, t):
        self.frontier += t
        self.n_spec = [s + t for s in self.n_spec]


class RollingAcceptance:
    """Fixed window of per-round acceptance rates (caches.py:655-674)."""

    def __init__(self, window: int):
        if window < 1:
            raise ValueError("window must be >= 1")
        self.window = window
        self.rates: list = []

    def push(self, rate: float):
        self.rates.append(float(rate))
        if len(self.rates) > self.window:
            self.rates.pop(0)

    @property
    def full(self) -> bool:
        return len(self.rates) >= self.window

    def mean(self) -> float:
        return float(np.mean(self.rates)) if self.rates else 1.0


def should_rebuild(config: RetrievalConfig, tokens_since_build: int, rolling: RollingAcceptance) -> bool:
    """Rebuild at the stride, or when a full window's mean acceptance drops
    below the threshold (caches.py:677-683)."""
    if tokens_since_build >= config.rebuild_stride:
        return True
    return rolling.full and rolling.mean() < config.rebuild_accept_threshold
