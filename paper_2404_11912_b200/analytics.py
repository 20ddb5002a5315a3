"""Acceptance-rate measurement over a prompt corpus on the device path --
the GPU counterpart of hierspec/analytics.py:229-309 (`AcceptanceStats`,
`measure_acceptance`).

Pairings: 'hierarchical' (draft model + StreamingCache speculated against
the retrieval-cache target, verified on the full cache; both levels are
reported) and the self-speculation pairings 'self:streaming',
'self:retrieval', 'self:topk' and 'self:h2o' (SingleLevelSession against the
full cache; TopK selects per layer and query on the device, csrc/topk.cu;
H2O feeds back the forward's attention probabilities, csrc/h2o.cu).
The rest of the reference's analytics module (attention-mass recovery,
needle fixtures, the speedup model) is host-side analysis, not decode work.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

from .caches import H2OCache, H2OConfig, RetrievalCache, RetrievalConfig, StreamingCache, StreamingConfig, TopKCache
from .model import ModelConfig, ModelWeights
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
