"""Hierarchical speculative decoding on B200 -- the drop-in for
hierspec/speculation.py (Algorithm 1 of TriForce).

Structure of one outer round (speculation.py:338-368):
  draft lane (StreamingCache)  -> gamma1 drafted tokens per inner round
  retrieval lane (RetrievalCache) scores them, verify chain -> x_hat
  ... until len(x_hat) >= gamma2
  full lane (FullCache) scores x_hat in ONE batched forward, verify chain.

Device residency: drafted tokens, draft/target distributions (fp64 [rows, V])
and the uniforms stay on the device; the host reads back only the few
emitted token ids, the accepted count and the RNG cursor once per inner and
once per outer round (it needs them for its control flow).  The RNG
protocol -- one uniform per draft sample, one per verification, one per
correction/bonus, in loop order from one PCG64 stream -- is the
reference's (speculation.py:9-12), so traces replay the CPU engine.
"""

from __future__ import annotations

import ctypes as C
import gc
import json
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from ._abi import check, lib, status_error
from .caches import (FullCache, H2OCache, KVCache, RetrievalCache, RetrievalConfig, RollingAcceptance, StreamingCache,
                     StreamingConfig, should_rebuild)
from .errors import ContractError
from .model import ForwardRecorder, ModelWeights, forward_device
from .runtime import STATS, UniformStream, as_device_f64, device, ptr, staging, stream_ptr, to_i32_device

# CUDA-graph replay of the draft lane's one-token steps (HS_NO_GRAPHS=1 turns
# it off: every step is then a regular hs_forward call with the same kernels)
USE_GRAPHS = os.environ.get("HS_NO_GRAPHS", "0") != "1"

# NVTX ranges per lane and phase (HS_NVTX=1): rebuild, inner round (draft
# round, retrieval score, verify chain), outer verify -- visible in nsys / ncu
# --nvtx timelines.  Off by default (a range push/pop costs ~1 us of host time).
USE_NVTX = os.environ.get("HS_NVTX", "0") == "1"


class _nvtx:
    __slots__ = ("name",)

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        if USE_NVTX:
            torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *exc):
        if USE_NVTX:
            torch.cuda.nvtx.range_pop()


class _StepGraph:
    """One-token forward of a streaming-cache lane captured as a CUDA graph.

    The draft model is tiny (JF68M shape: 2 layers), so its step is bound by
    the host launching ~25 kernels, not by the GPU.  The graph reads its
    token from a fixed device slot and the frontier / window watermark from a
    device int32[2] (HsStep.dyn) refreshed before each replay, so one capture
    serves every position.  It keeps references to every buffer it was
    captured with (workspace, logits rows) so later re-allocations elsewhere
    cannot invalidate it."""

    def __init__(self, lane: "Lane"):
        cache = lane.cache
        dm = lane.weights.device()
        cfg = dm.config
        self.lane = lane
        # [frontier, window watermark, token]: one fixed device slot the graph
        # reads its positions and its input token from
        self.dyn = torch.zeros(3, dtype=torch.int32, device=device())
        self.tok = tok = self.dyn[2:3]
        step = cache._step(1)
        step.pos0, step.win_lo, step.dyn = 0, 0, self.dyn.data_ptr()
        self.step = step
        self.nbytes = lib.hs_forward_workspace_bytes(dm.ref, 1, step.n_view, step.split, 0)
        self.ws = dm.workspace(self.nbytes)
        self.out = torch.empty((1, cfg.vocab_size), dtype=torch.float32, device=device())
        self.stash = lane.recorder._buffer(cfg)
        self.alg_bytes = dm.weight_bytes + step.n_view * cfg.n_kv_heads * cfg.head_dim * 4 * cfg.n_layers
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        n0 = lib.hs_launch_count()
        # capture_begin/end directly (torch.cuda.graph's context manager
        # synchronises the whole device first); thread_local: other host
        # threads (loopback shard ranks) keep launching on their own streams
        # while this one captures
        # (a graph object freed by the cycle collector during the capture
        # would destroy its executable mid-capture and invalidate it: keep the
        # collector off until the capture ends; nothing in the captured region
        # drops a reference to a graph)
        was_enabled = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.stream(side):
                self.graph.capture_begin(capture_error_mode="thread_local")
                try:
                    check(lib.hs_forward(dm.ref, cache._ref, C.byref(step), None, ptr(tok), 1, ptr(self.out),
                                         ptr(self.stash), ptr(self.ws), self.nbytes, stream_ptr()))
                    lane._front.copy_(self.out[0])
                finally:
                    self.graph.capture_end()
        finally:
            if was_enabled:
                gc.enable()
        self.n_launch = lib.hs_launch_count() - n0
        torch.cuda.current_stream().wait_stream(side)
        # the executable graph, launched natively (hs_draft_step / hs_graph_step)
        # right after the kernel that writes its positions -- no staging copy
        self.exec = C.c_void_p(int(self.graph.raw_cuda_graph_exec()))
        self.dyn_ptr = self.dyn.data_ptr()

    def prep(self):
        """Host checks of one step on the live state; its positions."""
        cache = self.lane.cache
        cache._guard(cache.frontier, cache.frontier)     # the ring keeps every exposable entry
        return cache.frontier, cache.lo

    def post(self) -> None:
        lane, cache = self.lane, self.lane.cache
        STATS["alg_bytes"] += self.alg_bytes
        cache._advance(1)
        lane._has_front = True
        lane.recorder.query_position = cache.frontier - 1

    def run(self, host_token: Optional[int] = None, also=None) -> None:
        """One step; the token is already in self.tok (device) or is
        host_token (written with the positions by one tiny kernel, and also
        to the device int32 `also` when given)."""
        f, lo = self.prep()
        check(lib.hs_graph_step(self.dyn_ptr, f, lo, -1 if host_token is None else int(host_token),
                                also, self.exec, self.n_launch, stream_ptr()))
        self.post()



# process-wide counters (bench.py reads them around its timed region)
COUNTERS = {"inner_rounds": 0, "inner_proposed": 0, "inner_accepted": 0, "outer_rounds": 0, "outer_proposed": 0,
            "outer_accepted": 0, "rebuilds": 0, "h2d_bytes": 0, "d2h_bytes": 0}


@dataclass
class SpecConfig:
    """Algorithm 1 parameters (speculation.py:35-49)."""
    target_len: int
    gamma1: int = 2
    gamma2: int = 6
    temperature: float = 0.0
    seed: int = 0
    streaming: StreamingConfig = field(default_factory=StreamingConfig)
    retrieval: RetrievalConfig = field(default_factory=RetrievalConfig)

    def __post_init__(self):
        if self.gamma1 < 1 or self.gamma2 < 1:
            raise ValueError("gamma1 and gamma2 must be >= 1")
        if self.temperature < 0:
            raise ValueError("temperature must be >= 0")


class _Cat:
    """committed + x_hat without copying the (100K+ token) committed list:
    lanes only take len() and a tail slice of the sequence."""

    __slots__ = ("head", "tail")

    def __init__(self, head, tail):
        self.head, self.tail = head, tail

    def __len__(self):
        return len(self.head) + len(self.tail)

    def __getitem__(self, sl):
        if not isinstance(sl, slice) or sl.step not in (None, 1) or sl.stop is not None:
            raise TypeError("_Cat supports tail slices only")
        a = sl.start or 0
        n = len(self.head)
        return (list(self.head[a:]) if a < n else []) + list(self.tail[max(0, a - n):])


def _one_uniform(rng) -> tuple:
    u = torch.tensor([rng.random()], dtype=torch.float64, device=device())
    cur = torch.zeros(1, dtype=torch.int32, device=u.device)
    return u, cur


def verify_token(x: int, q, p, rng: np.random.Generator) -> bool:
    """Accept x ~ q with probability min(1, p[x]/q[x]); one uniform
    (speculation.py:52-62).  q[x] <= 0 raises ContractError."""
    qd, pd = as_device_f64(q).reshape(-1), as_device_f64(p).reshape(-1)
    if float(qd[int(x)].item()) <= 0.0:
        raise ContractError(f"verify_token: draft distribution assigns 0 to token {x}")
    u, cur = _one_uniform(rng)
    res = torch.zeros(2, dtype=torch.int32, device=u.device)
    check(lib.hs_verify_token(int(x), ptr(qd), ptr(pd), ptr(u), ptr(cur), ptr(res), stream_ptr()))
    return bool(res[0].item())


def correct_token(q, p, rng: np.random.Generator) -> int:
    """Sample normalize(max(p - q, 0)), falling back to p when the residual
    vanishes; one uniform (speculation.py:65-72)."""
    qd, pd = as_device_f64(q).reshape(-1), as_device_f64(p).reshape(-1)
    u, cur = _one_uniform(rng)
    out = torch.zeros(1, dtype=torch.int32, device=u.device)
    check(lib.hs_correct_token(ptr(qd), ptr(pd), pd.numel(), ptr(u), ptr(cur), ptr(out), stream_ptr()))
    return int(out.item())


class Lane:
    """Model + cache + frontier logits row (speculation.py:75-130).  The
    frontier row lives in a device buffer; `None` semantics are tracked on
    the host."""

    def __init__(self, weights: ModelWeights, cache: KVCache):
        self.weights = weights
        self.cache = cache
        self.recorder = ForwardRecorder(record_probs=False)
        V = weights.config.vocab_size
        self._front = torch.zeros(V, dtype=torch.float32, device=device())
        self._has_front = False
        self._scratch = None
        self._graph = None
        # shard.SequenceShards splitting this lane's dense projections
        # (tensor parallel, hs_forward_tp); None = replicated weights
        self.tp = None

    def step_graph(self) -> "_StepGraph":
        if self._graph is None:
            self._graph = _StepGraph(self)
        return self._graph

    def step_graph_run(self, tok, also=None) -> None:
        """One-token step through the lane's captured graph.  The graph reads
        its token from a lane-owned device slot (one capture per lane, never
        per caller buffer); a device `tok` is copied into it on the stream, a
        host int travels with the step's positions (and is also written to
        the device int32 address `also`)."""
        g = self.step_graph()
        if isinstance(tok, torch.Tensor):
            g.tok.copy_(tok)
            g.run()
        else:
            g.run(host_token=int(tok), also=also)

    @property
    def frontier(self) -> int:
        return self.cache.frontier

    @property
    def frontier_logits(self):
        return self._front if self._has_front else None

    @frontier_logits.setter
    def frontier_logits(self, value):
        if value is None:
            self._has_front = False
        else:
            self._front.copy_(torch.as_tensor(value, dtype=torch.float32).reshape(-1).to(self._front.device))
            self._has_front = True

    def _logits_buf(self, t: int) -> torch.Tensor:
        V = self.weights.config.vocab_size
        if self._scratch is None or self._scratch.shape[0] < t:
            self._scratch = torch.empty((max(t, 16), V), dtype=torch.float32, device=device())
        return self._scratch[:t]

    def _forward(self, tokens) -> torch.Tensor:
        """Forward (host list or device int32 tensor) -> device logits [t, V];
        updates the frontier row."""
        t = tokens.numel() if isinstance(tokens, torch.Tensor) else len(tokens)
        out = forward_device(self.weights, tokens, self.cache, self.recorder, out=self._logits_buf(t), tp=self.tp)
        self._front.copy_(out[t - 1])
        self._has_front = True
        return out

    def prefill(self, tokens: Sequence[int]) -> None:
        if len(tokens) == 0:
            raise ValueError("prefill needs at least one token")
        t = len(tokens)
        out = forward_device(self.weights, list(tokens), self.cache, self.recorder, out=self._logits_buf(t),
                             prefill=True)
        self._front.copy_(out[t - 1])
        self._has_front = True
        self.cache.commit(self.cache.frontier)

    def advance(self, tokens: Sequence[int]) -> None:
        if len(tokens):
            self._forward(list(tokens))

    def catch_up(self, sequence: Sequence[int]) -> None:
        if self.frontier < len(sequence):
            self.advance(list(sequence[self.frontier:]))

    def score(self, tokens: Sequence[int]) -> list:
        """len(tokens) + 1 logits rows (device), the first being the current
        frontier row -- one batched forward."""
        if not self._has_front:
            raise ContractError("lane has no frontier logits; advance over committed tokens first")
        rows = [self._front.clone()]
        if len(tokens):
            out = self._forward(list(tokens))
            rows.extend(out[i].clone() for i in range(out.shape[0]))
        return rows

    def rollback_to(self, n: int) -> None:
        if n < self.cache.frontier:
            self._has_front = False
        self.cache.rollback_to(n)

    def commit(self) -> None:
        self.cache.commit(self.cache.frontier)

    def last_queries(self) -> list:
        return self.recorder.last_queries

    def clone(self) -> "Lane":
        c = Lane(self.weights, self.cache.clone())
        c.tp = self.tp
        c._front.copy_(self._front)
        c._has_front = self._has_front
        if self.recorder.stash is not None:
            c.recorder.stash = self.recorder.stash.clone()
        return c


@dataclass
class LevelStats:
    proposed: int = 0
    accepted: int = 0
    rounds: int = 0

    @property
    def rejected(self) -> int:
        return self.proposed - self.accepted

    @property
    def rate(self) -> float:
        return self.accepted / self.proposed if self.proposed else 0.0


class StepTrace:
    """Per-token provenance, JSON-lines serialisable (speculation.py:148-184)."""

    def __init__(self):
        self.records: list = []
        self.inner = LevelStats()
        self.outer = LevelStats()

    def add(self, position, token, level, accepted, outer_round):
        self.records.append({"position": int(position), "token": int(token), "level": level,
                             "accepted": bool(accepted), "outer_round": int(outer_round)})

    def truncate(self, n_tokens: int):
        self.records = self.records[:n_tokens]

    def emitted_tokens(self) -> list:
        return [r["token"] for r in self.records]

    def to_jsonl(self, fp) -> None:
        for r in self.records:
            fp.write(json.dumps(r) + "\n")

    def summary(self) -> dict:
        def lv(s):
            return {"proposed": s.proposed, "accepted": s.accepted, "rounds": s.rounds, "rate": s.rate}
        return {"emitted": len(self.records), "inner": lv(self.inner), "outer": lv(self.outer)}


# ---------------------------------------------------------------------------
# device round machinery

class _RoundBuffers:
    def __init__(self, V: int, gamma1: int, gamma2: int):
        dev = device()
        rows = gamma1 + gamma2 + 2
        self.V = V
        self.q = torch.empty((gamma1, V), dtype=torch.float64, device=dev)
        self.dtok = torch.empty(gamma1, dtype=torch.int32, device=dev)
        self.p = torch.empty((rows, V), dtype=torch.float64, device=dev)
        self.phat = torch.empty((rows, V), dtype=torch.float64, device=dev)
        self.xtok = torch.empty(rows, dtype=torch.int32, device=dev)
        # retrieval-lane input of an inner round whose catch-up is 1-2 tokens:
        # [catch-up tokens, drafted tokens...] -- written in place by the draft
        # lane's steps, so the retrieval forward needs no concatenation
        self.rtok = torch.empty(gamma1 + 2, dtype=torch.int32, device=dev)
        # the full lane's input of an outer round: [catch-up tokens, x_hat]
        self.ftok = torch.empty(rows + 2, dtype=torch.int32, device=dev)
        self.res = torch.zeros(rows + 4, dtype=torch.int32, device=dev)
        self.host = torch.zeros(rows + 5, dtype=torch.int32, pin_memory=True)


def _readback(buf: _RoundBuffers, n: int, us: UniformStream):
    """One device->host sync: chain result for n proposals + RNG cursor."""
    buf.host[:n + 4].copy_(buf.res[:n + 4], non_blocking=True)
    buf.host[n + 4:n + 5].copy_(us.cursor, non_blocking=True)
    check(lib.hs_stream_sync(stream_ptr()))
    COUNTERS["d2h_bytes"] += 4 * (n + 5)
    h = buf.host.numpy()
    count, accepted, status, cursor = int(h[n + 1]), int(h[n + 2]), int(h[n + 3]), int(h[n + 4])
    if status != 0:
        raise status_error(status, "verify_token: draft distribution assigns 0 to the drafted token")
    return [int(x) for x in h[:count]], accepted, cursor


def _draft_round_dev(lane: Lane, seq: Sequence[int], gamma1: int, T: float, us: UniformStream,
                     buf: _RoundBuffers, fused: int = 0) -> torch.Tensor:
    """draft_round (speculation.py:211-227) with tokens and q rows on device;
    returns the device tensor holding the drafted tokens.  fused = k > 0: the
    lane's catch-up is the last k tokens of seq, also written to buf.rtok[:k],
    and the drafts go to buf.rtok[k:] (the retrieval lane's whole input, in
    place)."""
    graphs = USE_GRAPHS and isinstance(lane.cache, StreamingCache)
    k = len(seq) - lane.frontier
    fused = fused if (fused and graphs and k == fused) else 0
    if graphs and 1 <= k <= 2:
        # the usual one- or two-token catch-up, one graph step per token
        rp = buf.rtok.data_ptr()
        tail = list(seq[len(seq) - k:])
        for i in range(k):
            lane.step_graph_run(tail[i], also=rp + 4 * i if fused else None)
    else:
        lane.catch_up(seq)
    if not lane._has_front:
        raise ContractError("lane has no frontier logits; advance over committed tokens first")
    V = buf.V
    s = stream_ptr()
    dtok = buf.rtok[fused:fused + gamma1] if fused else buf.dtok
    if graphs:
        # sample -> write token + positions into the step graph's slot -> graph,
        # one native call per drafted token
        sg = lane.step_graph()
        front, qp, tp = lane._front.data_ptr(), buf.q.data_ptr(), dtok.data_ptr()
        ub, uc = us.buf.data_ptr(), us.cursor.data_ptr()
        for g in range(gamma1):
            f, lo = sg.prep()
            check(lib.hs_draft_step(front, V, float(T), qp + 8 * V * g, ub, uc, tp + 4 * g, sg.dyn_ptr, f, lo,
                                    sg.exec, sg.n_launch, s))
            sg.post()
        return dtok
    for g in range(gamma1):
        check(lib.hs_draft_sample(ptr(lane._front), V, float(T), ptr(buf.q[g]), ptr(us.buf), ptr(us.cursor),
                                  ptr(dtok[g:g + 1]), s))
        lane._forward(dtok[g:g + 1])
    return dtok


def _score_rows_dev(lane: Lane, seq: Sequence[int], tokens_dev: torch.Tensor, T: float,
                    out: torch.Tensor) -> None:
    """lane.catch_up(seq) + lane.score(tokens) as ONE batched forward; the
    len(tokens)+1 target distributions go to out[0:n+1] (fp64)."""
    V = lane.weights.config.vocab_size
    s = stream_ptr()
    cu = list(seq[lane.frontier:])
    n = tokens_dev.numel()
    if not cu:
        if not lane._has_front:
            raise ContractError("lane has no frontier logits; advance over committed tokens first")
        check(lib.hs_probs(ptr(lane._front), 1, V, float(T), ptr(out[0]), s))
    toks = torch.cat([to_i32_device(cu), tokens_dev]) if cu else tokens_dev
    COUNTERS["h2d_bytes"] += 4 * len(cu)
    logits = lane._forward(toks)
    if cu:
        check(lib.hs_probs(ptr(logits[len(cu) - 1]), n + 1, V, float(T), ptr(out[0]), s))
    else:
        check(lib.hs_probs(ptr(logits[0]), n, V, float(T), ptr(out[1]), s))


def _chain_dev(tokens_dev, n, qd, pd, V, us, buf):
    check(lib.hs_verify_chain(ptr(tokens_dev), n, ptr(qd), ptr(pd), V, ptr(us.buf), ptr(us.cursor), ptr(buf.res),
                              stream_ptr()))


def _inner_round_dev(retr: Lane, draft: Lane, seq, cfg: SpecConfig, us, buf, phat_off: int):
    V = buf.V
    # both lanes sit at the same frontier: a one- (two-, after an all-accept
    # outer round) token catch-up is the usual case
    k = len(seq) - retr.frontier
    fused = k if (1 <= k <= 2 and draft.frontier == retr.frontier) else 0
    with _nvtx("inner.draft_round"):
        dtok = _draft_round_dev(draft, seq, cfg.gamma1, cfg.temperature, us, buf, fused=fused)
    with _nvtx("inner.retrieval_score"):
        if dtok.data_ptr() != buf.dtok.data_ptr():
            # buf.rtok = [catch-up, drafts]: one forward, rows k-1 .. k-1+gamma1
            n = cfg.gamma1
            logits = retr._forward(buf.rtok[:fused + n])
            check(lib.hs_probs(logits.data_ptr() + 4 * V * (fused - 1), n + 1, V, float(cfg.temperature),
                               buf.p.data_ptr(), stream_ptr()))
        else:
            _score_rows_dev(retr, seq, dtok, cfg.temperature, buf.p)
    with _nvtx("inner.verify_chain"):
        _chain_dev(dtok, cfg.gamma1, buf.q, buf.p, V, us, buf)
        # p_hat rows of the emitted tokens: copy all gamma1+1, the surplus is overwritten later
        buf.phat[phat_off:phat_off + cfg.gamma1 + 1].copy_(buf.p[:cfg.gamma1 + 1])
        return _readback(buf, cfg.gamma1, us)


# ---------------------------------------------------------------------------
# public single-round API (speculation.py:211-275) -- numpy in/out

def _api_buffers(lane: Lane, gamma1: int, gamma2: int) -> _RoundBuffers:
    return _RoundBuffers(lane.weights.config.vocab_size, gamma1, gamma2)


def draft_round(draft_lane: Lane, committed: Sequence[int], gamma1: int, temperature: float,
                rng: np.random.Generator):
    """Draft gamma1 tokens; returns (tokens, q distributions as numpy)."""
    us = UniformStream(rng, block=max(64, gamma1), keep_state=True)
    buf = _api_buffers(draft_lane, gamma1, 1)
    _draft_round_dev(draft_lane, list(committed), gamma1, temperature, us, buf)
    toks = buf.dtok.cpu().numpy().astype(int).tolist()
    us.sync_rng(gamma1)
    return toks, [buf.q[i].cpu().numpy() for i in range(gamma1)]


def _verify_chain(tokens, draft_dists, target_dists, rng):
    """(emitted, labels, accepted) -- speculation.py:187-208."""
    n = len(tokens)
    V = len(target_dists[0])
    us = UniformStream(rng, block=max(64, n + 1), keep_state=True)
    buf = _RoundBuffers(V, max(n, 1), max(n, 1))
    tok = to_i32_device(list(tokens)) if n else torch.zeros(1, dtype=torch.int32, device=device())
    qd = torch.stack([as_device_f64(x).reshape(-1) for x in draft_dists]) if n else buf.q
    pd = torch.stack([as_device_f64(x).reshape(-1) for x in target_dists])
    _chain_dev(tok, n, qd, pd, V, us, buf)
    emitted, accepted, cursor = _readback(buf, n, us)
    us.sync_rng(cursor)
    labels = ["accepted"] * accepted + (["corrected"] if accepted < n else ["bonus"])
    return emitted, labels, accepted


def inner_speculate(retr_lane: Lane, draft_lane: Lane, committed: Sequence[int], config: SpecConfig,
                    rng: np.random.Generator, trace: Optional[StepTrace] = None):
    """Draft rounds verified against the retrieval lane until >= gamma2
    tokens (speculation.py:230-261).  Returns (x_hat, p_hats, labels)."""
    V = retr_lane.weights.config.vocab_size
    us = UniformStream(rng, keep_state=True)
    buf = _RoundBuffers(V, config.gamma1, config.gamma2)
    x_hat, labels, cursor = [], [], 0
    base = len(committed)
    while len(x_hat) < config.gamma2:
        us.ensure(2 * config.gamma1 + 2, cursor)
        emitted, accepted, cursor = _inner_round_dev(retr_lane, draft_lane, _Cat(committed, x_hat), config, us,
                                                     buf, len(x_hat))
        x_hat.extend(emitted)
        labels.extend(["draft"] * accepted + ["retrieval"])
        if trace is not None:
            trace.inner.rounds += 1
            trace.inner.proposed += config.gamma1
            trace.inner.accepted += accepted
        valid = base + len(x_hat) - 1
        draft_lane.rollback_to(valid)
        retr_lane.rollback_to(valid)
    us.sync_rng(cursor)
    return x_hat, [buf.phat[i].cpu().numpy() for i in range(len(x_hat))], labels


def outer_verify(full_lane: Lane, committed: Sequence[int], x_hat: Sequence[int], p_hats, temperature: float,
                 rng: np.random.Generator):
    """Score x_hat under the full cache (one batched forward) and verify
    (speculation.py:264-275).  Returns (emitted, labels, accepted, pdists)."""
    n = len(x_hat)
    V = full_lane.weights.config.vocab_size
    us = UniformStream(rng, block=max(64, n + 1), keep_state=True)
    buf = _RoundBuffers(V, 1, n)
    xt = to_i32_device(list(x_hat))
    _score_rows_dev(full_lane, list(committed), xt, temperature, buf.p)
    qd = torch.stack([as_device_f64(x).reshape(-1) for x in p_hats])
    _chain_dev(xt, n, qd, buf.p, V, us, buf)
    emitted, accepted, cursor = _readback(buf, n, us)
    us.sync_rng(cursor)
    labels = ["accepted"] * accepted + (["corrected"] if accepted < n else ["bonus"])
    return emitted, labels, accepted, [buf.p[i].cpu().numpy() for i in range(n + 1)]


# ---------------------------------------------------------------------------
# the two-level session

class HierarchicalSession:
    """Prefilled lanes for one (target, draft, prefix) triple
    (speculation.py:278-368).  Single-threaded; clone() snapshots."""

    def __init__(self, target: ModelWeights, draft: ModelWeights, prefix: Sequence[int], config: SpecConfig,
                 _prefill: bool = True, shards=None, tp=None):
        """shards: a shard.SequenceShards -- the full cache is then split
        along the sequence over its ranks (every rank runs this session with
        the same arguments).  None = one GPU.
        tp: a shard.SequenceShards (typically the same object) over which the
        target's dense projections of the full and retrieval lanes are split
        by output rows (tensor parallel); the draft lane
        stays replicated."""
        if target.config.vocab_size != draft.config.vocab_size:
            raise ContractError("target and draft models must share a vocabulary")
        if len(prefix) < 1:
            raise ValueError("prefix must be non-empty")
        if config.target_len <= len(prefix):
            raise ValueError("target_len must exceed the prefix length")
        self.config = config
        self.committed = list(prefix)
        full = (FullCache.from_config(target.config) if shards is None else
                FullCache.shard(target.config, shards, len(prefix), config.retrieval.chunk_size))
        self.full_lane = Lane(target, full)
        self.draft_lane = Lane(draft, StreamingCache.from_config(draft.config, config.streaming))
        self.retr_lane = Lane(target, RetrievalCache.from_config(target.config, config.retrieval))
        self.full_lane.tp = self.retr_lane.tp = tp
        self.rolling = RollingAcceptance(config.retrieval.rolling_window)
        self.tokens_since_build = 0
        self.rebuilds = 0
        self._buf = _RoundBuffers(target.config.vocab_size, config.gamma1, config.gamma2)
        if _prefill:
            self.full_lane.prefill(prefix)
            self.draft_lane.prefill(prefix)
            self._initial_build()

    def _initial_build(self):
        n = len(self.committed)
        retr: RetrievalCache = self.retr_lane.cache
        q = self.full_lane.recorder.stash
        if n >= 2:
            retr.build(self.full_lane.cache, q, upto=n - 1)
        else:
            retr.build(self.full_lane.cache, q, upto=n)
            self.retr_lane.frontier_logits = self.full_lane.frontier_logits

    @classmethod
    def synthetic(cls, target: ModelWeights, draft: ModelWeights, context: Sequence[int], config: SpecConfig,
                  seed: int = 0, shards=None, tp=None):
        """Session over a synthetic long context (throughput configs,
        SURVEY §7.4 item 6): the full and draft caches are filled with random
        bf16 K/V for positions [0, n-1); the last context token is then
        decoded for real on every lane and the initial build uses its queries."""
        s = cls(target, draft, context, config, _prefill=False, shards=shards, tp=tp)
        n = len(context)
        s.full_lane.cache.fill_random_(n - 1, seed=seed)
        s.draft_lane.cache.fill_random_(n - 1, seed=seed + 1)
        s.full_lane.advance([context[-1]])
        s.full_lane.commit()
        s.draft_lane.advance([context[-1]])
        s.draft_lane.commit()
        s._initial_build()
        return s

    def clone(self) -> "HierarchicalSession":
        c = object.__new__(HierarchicalSession)
        c.config = self.config
        c.committed = list(self.committed)
        c.full_lane = self.full_lane.clone()
        c.draft_lane = self.draft_lane.clone()
        c.retr_lane = self.retr_lane.clone()
        c.rolling = RollingAcceptance(self.config.retrieval.rolling_window)
        c.rolling.rates = list(self.rolling.rates)
        c.tokens_since_build = self.tokens_since_build
        c.rebuilds = self.rebuilds
        c._buf = _RoundBuffers(self.full_lane.weights.config.vocab_size, self.config.gamma1, self.config.gamma2)
        return c

    def _maybe_rebuild(self) -> bool:
        cache: RetrievalCache = self.retr_lane.cache
        if not should_rebuild(cache.config, self.tokens_since_build, self.rolling):
            return False
        # queries of the last committed token under the OLD exposure
        # (speculation.py:324-336), then rebuild from the full cache
        self.retr_lane.catch_up(self.committed)
        cache.build(self.full_lane.cache, self.retr_lane.recorder.stash, upto=self.full_lane.frontier)
        self.retr_lane.frontier_logits = None
        self.tokens_since_build = 0
        self.rolling.rates.clear()
        self.rebuilds += 1
        COUNTERS["rebuilds"] += 1
        return True

    def generate(self, seed: Optional[int] = None):
        """Run the two-level loop until target_len tokens are committed;
        returns (tokens, StepTrace)."""
        cfg = self.config
        rng = np.random.default_rng(cfg.seed if seed is None else seed)
        us = UniformStream(rng)
        buf = self._buf
        trace = StepTrace()
        cursor = 0
        V = buf.V
        while len(self.committed) < cfg.target_len:
            with _nvtx("rebuild_check"):
                self._maybe_rebuild()
            # ---- inner level: draft -> retrieval (speculation.py:230-261)
            x_hat, ilabels = [], []
            base = len(self.committed)
            while len(x_hat) < cfg.gamma2:
                us.ensure(2 * cfg.gamma1 + 2, cursor)
                emitted, accepted, cursor = _inner_round_dev(self.retr_lane, self.draft_lane,
                                                             _Cat(self.committed, x_hat), cfg, us, buf, len(x_hat))
                x_hat.extend(emitted)
                ilabels.extend(["draft"] * accepted + ["retrieval"])
                trace.inner.rounds += 1
                trace.inner.proposed += cfg.gamma1
                trace.inner.accepted += accepted
                COUNTERS["inner_rounds"] += 1
                COUNTERS["inner_proposed"] += cfg.gamma1
                COUNTERS["inner_accepted"] += accepted
                valid = base + len(x_hat) - 1
                self.draft_lane.rollback_to(valid)
                self.retr_lane.rollback_to(valid)
            # ---- outer level: full-cache verify (speculation.py:264-275)
            n = len(x_hat)
            us.ensure(n + 2, cursor)
            with _nvtx("outer.verify"):
                # [catch-up, x_hat] in one upload, one forward
                full = self.full_lane
                cu = self.committed[full.frontier:]
                k = len(cu)
                toks = np.asarray(cu + x_hat, dtype=np.int32)
                s = stream_ptr()
                check(lib.hs_upload_i32(buf.ftok.data_ptr(), toks.ctypes.data, k + n, s))
                COUNTERS["h2d_bytes"] += 4 * (k + n)
                if k:
                    logits = full._forward(buf.ftok[:k + n])
                    check(lib.hs_probs(logits.data_ptr() + 4 * V * (k - 1), n + 1, V, float(cfg.temperature),
                                       buf.p.data_ptr(), s))
                else:
                    if not full._has_front:
                        raise ContractError("lane has no frontier logits; advance over committed tokens first")
                    check(lib.hs_probs(full._front.data_ptr(), 1, V, float(cfg.temperature), buf.p.data_ptr(), s))
                    logits = full._forward(buf.ftok[:n])
                    check(lib.hs_probs(logits.data_ptr(), n, V, float(cfg.temperature), buf.p.data_ptr() + 8 * V, s))
                xt = buf.ftok[k:k + n]
                _chain_dev(xt, n, buf.phat, buf.p, V, us, buf)
                emitted, accepted, cursor = _readback(buf, n, us)
            olabels = ["accepted"] * accepted + (["corrected"] if accepted < n else ["bonus"])
            trace.outer.rounds += 1
            trace.outer.proposed += n
            trace.outer.accepted += accepted
            COUNTERS["outer_rounds"] += 1
            COUNTERS["outer_proposed"] += n
            COUNTERS["outer_accepted"] += accepted
            emitted = emitted[:cfg.target_len - base]
            for i, tok in enumerate(emitted):
                level = ilabels[i] if olabels[i] == "accepted" else olabels[i]
                trace.add(base + i, tok, level, olabels[i] == "accepted", trace.outer.rounds)
            self.committed.extend(emitted)
            valid = base + min(accepted, len(emitted))
            if valid == len(self.committed):
                # truncated final round: the reference ends the session here with
                # lanes that hold every token but no frontier row; keep the last
                # token unprocessed instead so a later generate() can catch up
                valid -= 1
            self.full_lane.rollback_to(valid)
            self.full_lane.commit()
            for lane in (self.draft_lane, self.retr_lane):
                lane.rollback_to(min(lane.frontier, valid))
                lane.commit()
            self.rolling.push(accepted / n)
            self.tokens_since_build += len(emitted)
        return list(self.committed), trace


def hierarchical_generate(target: ModelWeights, draft: ModelWeights, prefix: Sequence[int], config: SpecConfig):
    """Two-level speculative generation (speculation.py:371-375)."""
    return HierarchicalSession(target, draft, prefix, config).generate()


def autoregressive_generate(weights: ModelWeights, prefix: Sequence[int], target_len: int,
                            temperature: float = 0.0, seed: int = 0, shards=None, chunk: int = 16,
                            tp=None) -> list:
    """Plain decode over the full cache (speculation.py:378-398); the
    sampled token never leaves the device until the end.  shards: sequence-
    shard the full cache (shard.SequenceShards, boundaries aligned to chunk)."""
    if len(prefix) < 1:
        raise ValueError("prefix must be non-empty")
    if target_len <= len(prefix):
        raise ValueError("target_len must exceed the prefix length")
    rng = np.random.default_rng(seed)
    cache = (FullCache.from_config(weights.config) if shards is None else
             FullCache.shard(weights.config, shards, len(prefix), chunk))
    lane = Lane(weights, cache)
    lane.tp = tp
    lane.prefill(list(prefix))
    return _ar_loop(lane, list(prefix), target_len, temperature, rng)


def _ar_loop(lane: Lane, out: list, target_len: int, temperature: float, rng) -> list:
    V = lane.weights.config.vocab_size
    n_new = target_len - len(out)
    us = UniformStream(rng, block=max(64, n_new))
    toks = torch.empty(n_new, dtype=torch.int32, device=device())
    probs = torch.empty(V, dtype=torch.float64, device=device())
    s = stream_ptr()
    for i in range(n_new):
        check(lib.hs_draft_sample(ptr(lane._front), V, float(temperature), ptr(probs), ptr(us.buf), ptr(us.cursor),
                                  ptr(toks[i:i + 1]), s))
        if i == n_new - 1:
            break
        lane._forward(toks[i:i + 1])
        lane.commit()
    return out + toks.cpu().numpy().astype(int).tolist()


class SingleLevelSession:
    """One draft lane speculated against one full-cache verify lane --
    standard speculative decoding, the acceptance-measurement pairing of
    speculation.py:401-477.  The draft cache is a StreamingCache (own draft
    model or self-speculation), a FullCache, TopKCache or H2OCache, or a
    RetrievalCache, which is built from (and rebuilt against) the verify
    lane's full cache and so requires the verify weights (self-speculation).
    Runs on the same device round machinery as HierarchicalSession: tokens,
    distributions and uniforms stay resident, one host read-back per round
    (an H2O draft also reads back its attention probabilities)."""

    def __init__(self, draft_weights: ModelWeights, draft_cache: KVCache, verify_weights: ModelWeights,
                 prefix: Sequence[int], gamma: int, temperature: float,
                 retrieval_config: Optional[RetrievalConfig] = None):
        if draft_weights.config.vocab_size != verify_weights.config.vocab_size:
            raise ContractError("draft and verify models must share a vocabulary")
        if gamma < 1:
            raise ValueError("gamma must be >= 1")
        if not isinstance(draft_cache, (FullCache, StreamingCache, RetrievalCache, H2OCache)):
            raise ContractError(f"draft cache {type(draft_cache).__name__} is not supported on the device path "
                                "(full, streaming, retrieval, top-k or H2O caches)")
        self.gamma = gamma
        self.temperature = temperature
        self.committed = list(prefix)
        self.verify_lane = Lane(verify_weights, FullCache.from_config(verify_weights.config))
        self.draft_lane = Lane(draft_weights, draft_cache)
        self.verify_lane.prefill(prefix)
        self._retrieval = isinstance(draft_cache, RetrievalCache)
        self._buf = _RoundBuffers(verify_weights.config.vocab_size, gamma, 1)
        if self._retrieval:
            if draft_weights is not verify_weights:
                raise ContractError("retrieval drafting requires shared weights (self-speculation)")
            n = len(prefix)
            draft_cache.build(self.verify_lane.cache, self.verify_lane.recorder.stash, upto=max(n - 1, 1))
            if n < 2:
                self.draft_lane.frontier_logits = self.verify_lane.frontier_logits
            self.rolling = RollingAcceptance(draft_cache.config.rolling_window)
            self.tokens_since_build = 0
        else:
            self.draft_lane.prefill(prefix)

    def _maybe_rebuild(self) -> None:
        cache: RetrievalCache = self.draft_lane.cache
        if not should_rebuild(cache.config, self.tokens_since_build, self.rolling):
            return
        self.draft_lane.catch_up(self.committed)
        cache.build(self.verify_lane.cache, self.draft_lane.recorder.stash, upto=self.verify_lane.frontier)
        self.draft_lane.frontier_logits = None
        self.tokens_since_build = 0
        self.rolling.rates.clear()
        COUNTERS["rebuilds"] += 1

    def generate(self, target_len: int, seed: int = 0):
        """Speculate until target_len tokens are committed; returns
        (tokens, LevelStats)."""
        if target_len <= len(self.committed):
            raise ValueError("target_len must exceed the prefix length")
        rng = np.random.default_rng(seed)
        us = UniformStream(rng)
        buf, g, T = self._buf, self.gamma, self.temperature
        stats = LevelStats()
        cursor = 0
        while len(self.committed) < target_len:
            if self._retrieval:
                self._maybe_rebuild()
            us.ensure(2 * g + 2, cursor)
            _draft_round_dev(self.draft_lane, self.committed, g, T, us, buf)
            _score_rows_dev(self.verify_lane, self.committed, buf.dtok, T, buf.p)
            _chain_dev(buf.dtok, g, buf.q, buf.p, buf.V, us, buf)
            emitted, accepted, cursor = _readback(buf, g, us)
            stats.rounds += 1
            stats.proposed += g
            stats.accepted += accepted
            base = len(self.committed)
            self.committed.extend(emitted)
            valid = base + len(emitted) - 1
            for lane in (self.verify_lane, self.draft_lane):
                lane.rollback_to(min(lane.frontier, valid))
                lane.commit()
            if self._retrieval:
                self.rolling.push(accepted / g)
                self.tokens_since_build += len(emitted)
        del self.committed[target_len:]
        return list(self.committed), stats
