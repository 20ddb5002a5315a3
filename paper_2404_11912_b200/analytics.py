"""Acceptance-rate measurement over a prompt corpus on the device path --
the GPU counterpart of hierspec/analytics.py:229-309 (`AcceptanceStats`,
`measure_acceptance`).

Pairings: 'hierarchical' (draft model + StreamingCache speculated against
the retrieval-cache target, verified on the full cache; both levels are
reported) and the self-speculation pairings 'self:streaming',
'self:retrieval', 'self:topk' and 'self:h2o' (SingleLevelSession against the
full cache; TopK selects per layer and query on the device, csrc/topk.cu;
H2O feeds back the forward's attention probabilities, csrc/h2o.cu).
Attention-mass recovery (`sparsity_recovery`, `locality_recovery`) runs on
the device attention probes.  The needle fixtures and the host-side speedup
model live in host_analysis.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .caches import (FullCache, H2OCache, H2OConfig, RetrievalCache, RetrievalConfig, StreamingCache,
                     StreamingConfig, TopKCache)
from .model import (ForwardRecorder, ModelConfig, ModelWeights, decode_step, prefill, prob_from_logits,
                    sample_from_probs)
from .speculation import HierarchicalSession, LevelStats, SingleLevelSession, SpecConfig

SELF_PAIRINGS = ("self:streaming", "self:h2o", "self:retrieval", "self:topk")


@dataclass
class AcceptanceStats:
    """Pooled acceptance counts of one pairing (analytics.py:229-246)."""
    pairing: str
    proposed: int = 0
    accepted: int = 0
    rounds: int = 0
    per_case: list = field(default_factory=list)

    @property
    def rate(self) -> float:
        return self.accepted / self.proposed if self.proposed else 0.0

    def absorb(self, stats: LevelStats) -> None:
        self.proposed += stats.proposed
        self.accepted += stats.accepted
        self.rounds += stats.rounds
        self.per_case.append(stats.rate)


def _draft_cache_for(pairing: str, config: ModelConfig, *, streaming: StreamingConfig, h2o: H2OConfig,
                     retrieval: RetrievalConfig, topk_budget: int):
    """analytics.py:250-262 for the device cache kinds."""
    kind = pairing.split(":", 1)[1]
    if kind == "streaming":
        return StreamingCache.from_config(config, streaming)
    if kind == "retrieval":
        return RetrievalCache.from_config(config, retrieval)
    if kind == "topk":
        return TopKCache.from_config(config, topk_budget)
    if kind == "h2o":
        return H2OCache.from_config(config, h2o)
    raise ValueError(f"unknown pairing {pairing!r}")


def measure_acceptance(pairing: str, target: ModelWeights, prompts: Sequence[Sequence[int]], *,
                       draft: Optional[ModelWeights] = None, gamma: int = 4, temperature: float = 0.0,
                       gen_tokens: int = 16, seed: int = 0, streaming: StreamingConfig = StreamingConfig(),
                       h2o: H2OConfig = H2OConfig(), retrieval: RetrievalConfig = RetrievalConfig(),
                       topk_budget: int = 64, gamma2: int = 6) -> dict:
    """Aggregate acceptance rates for one speculation pairing over a corpus
    (analytics.py:265-309).  Per-case seeds are seed XOR case index."""
    if pairing == "hierarchical":
        if draft is None:
            raise ValueError("hierarchical pairing needs a draft model")
        inner = AcceptanceStats("hierarchical:inner")
        outer = AcceptanceStats("hierarchical:outer")
        for i, prompt in enumerate(prompts):
            cfg = SpecConfig(target_len=len(prompt) + gen_tokens, gamma1=gamma, gamma2=gamma2,
                             temperature=temperature, seed=seed ^ i, streaming=streaming, retrieval=retrieval)
            _, trace = HierarchicalSession(target, draft, prompt, cfg).generate()
            inner.absorb(trace.inner)
            outer.absorb(trace.outer)
        return {"inner": inner, "outer": outer}
    if pairing not in SELF_PAIRINGS:
        raise ValueError(f"unknown pairing {pairing!r}")
    stats = AcceptanceStats(pairing)
    for i, prompt in enumerate(prompts):
        cache = _draft_cache_for(pairing, target.config, streaming=streaming, h2o=h2o, retrieval=retrieval,
                                 topk_budget=topk_budget)
        session = SingleLevelSession(target, cache, target, prompt, gamma, temperature, retrieval_config=retrieval)
        _, s = session.generate(len(prompt) + gen_tokens, seed=seed ^ i)
        stats.absorb(s)
    return {"self": stats}


# ---------------------------------------------------------------------------
# attention-mass recovery (analytics.py:31-106) over the device probes
# (ForwardRecorder(record_probs=True) -> hs_forward_probe)

def _top_mass(row: np.ndarray, budget: int) -> float:
    """Mass of the `budget` largest weights of one attention row."""
    b = min(budget, row.shape[0])
    return float(np.sort(row.astype(np.float64))[::-1][:b].sum())


def sparsity_recovery(weights: ModelWeights, context_tokens: Sequence[int], budget: int) -> np.ndarray:
    """Per layer, the head-averaged attention mass of the final context query
    that its `budget` heaviest keys capture (analytics.py:36-48)."""
    cache = FullCache.from_config(weights.config)
    rec = ForwardRecorder(record_probs=True)
    prefill(weights, context_tokens, cache, rec)
    return np.array([np.mean([_top_mass(r, budget) for r in rows]) for rows in rec.last_probs], dtype=np.float64)


@dataclass
class LocalityCurves:
    """frozen[o, layer]: context-region mass captured by the key set frozen
    at the prefill query; fresh[o, layer]: a fresh top-k set's mass at offset
    o (analytics.py:51-61)."""
    budget: int
    frozen: np.ndarray
    fresh: np.ndarray


def locality_recovery(weights: ModelWeights, context_tokens: Sequence[int], budget: int, horizon: int,
                      temperature: float = 0.0, seed: int = 0) -> LocalityCurves:
    """How long the top-`budget` key set chosen by the last prefill query keeps
    capturing the attention of later decode queries (analytics.py:64-106)."""
    if horizon < 1:
        raise ValueError("horizon must be >= 1")
    cfg = weights.config
    cache = FullCache.from_config(cfg)
    rec = ForwardRecorder(record_probs=True)
    logits = prefill(weights, context_tokens, cache, rec)[-1]
    n_ctx = len(context_tokens)
    b = min(budget, n_ctx)
    # per layer / head: the prefill query's heaviest keys, ties to the lower position
    frozen_sets = [[np.lexsort((np.arange(n_ctx), -row.astype(np.float64)))[:b] for row in rows]
                   for rows in rec.last_probs]
    frozen = np.empty((horizon + 1, cfg.n_layers))
    fresh = np.empty_like(frozen)

    def record(o: int) -> None:
        for li, rows in enumerate(rec.last_probs):
            fz, fr = [], []
            for h, row in enumerate(rows):
                ctx = row[:n_ctx].astype(np.float64)
                tot = ctx.sum()
                fz.append(ctx[frozen_sets[li][h]].sum() / tot)
                fr.append(np.sort(ctx)[::-1][:b].sum() / tot)
            frozen[o, li] = np.mean(fz)
            fresh[o, li] = np.mean(fr)

    record(0)
    rng = np.random.default_rng(seed)
    for o in range(1, horizon + 1):
        tok = sample_from_probs(prob_from_logits(logits, temperature), rng)
        logits = decode_step(weights, tok, cache, rec)
        cache.commit(cache.frontier)
        record(o)
    return LocalityCurves(budget=b, frozen=frozen, fresh=fresh)
