"""Host-side analysis that accompanies the device path: the analytic and
Monte-Carlo speedup model of the two-level loop and the planted-needle
fixtures (the names of hierspec/analytics.py:109-226, 312-520).

None of this runs on the GPU or on the decode path -- it is arithmetic on
acceptance rates and latencies, and synthetic prompts / weights for the
acceptance experiments (`measure_acceptance`).  It is restated here from the
documented behaviour so that code written against the reference package's
API keeps working; the speedup model follows PAPER.md's round structure:

    inner phase   draft rounds of gamma1 proposals verified by the retrieval
                  lane, each round yielding k+1 tokens (k accepted, then a
                  correction) or gamma1+1 (all accepted + bonus), repeated
                  until at least gamma2 tokens are staged;
    outer phase   one full-cache verification of the staged n tokens,
                  committing expected_tokens(alpha2, n) of them.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from .model import BOS, ModelConfig, ModelWeights, generate_weights

DIGIT_TOKENS = tuple(range(ord("0"), ord("9") + 1))


# ---------------------------------------------------------------------------
# speedup model

def expected_tokens(alpha: float, gamma: int) -> float:
    """Mean tokens committed by one verification of `gamma` proposals, each
    accepted with probability alpha: 1 + alpha + ... + alpha^gamma."""
    if not 0.0 <= alpha <= 1.0:
        raise ValueError("alpha must be in [0, 1]")
    if gamma < 0:
        raise ValueError("gamma must be >= 0")
    return float(np.sum(alpha ** np.arange(gamma + 1, dtype=np.float64)))


@dataclass(frozen=True)
class LatencyModel:
    """Per-forward latencies (ms), affine in the tokens each forward attends."""
    draft_base: float = 0.5
    draft_per_token: float = 0.0005
    retrieval_base: float = 2.0
    retrieval_per_token: float = 0.002
    full_base: float = 2.0
    full_per_token: float = 0.006

    def __post_init__(self):
        for field_ in ("draft_base", "retrieval_base", "full_base"):
            if getattr(self, field_) <= 0:
                raise ValueError(f"{field_} must be positive")
        for field_ in ("draft_per_token", "retrieval_per_token", "full_per_token"):
            if getattr(self, field_) < 0:
                raise ValueError(f"{field_} must be non-negative")

    def t_draft(self, context: int, budget: int) -> float:
        return self.draft_base + self.draft_per_token * min(budget, context)

    def t_target_retrieval(self, context: int, budget: int) -> float:
        return self.retrieval_base + self.retrieval_per_token * min(budget, context)

    def t_target_full(self, context: int) -> float:
        return self.full_base + self.full_per_token * context

    def check(self, context: int, budget: int) -> None:
        if budget < context and self.t_target_full(context) < self.t_target_retrieval(context, budget):
            raise ValueError("full-cache forward must not be faster than the retrieval forward")


@dataclass
class SpeedupEstimate:
    tokens_per_round: float
    wall_ms_per_round: float
    speedup: float
    ci_halfwidth: float = 0.0
    inner_rounds_per_outer: float = 0.0


def _check_rates(alpha1, alpha2, gamma1, gamma2):
    if not (0.0 <= alpha1 <= 1.0 and 0.0 <= alpha2 <= 1.0):
        raise ValueError("acceptance rates must be in [0, 1]")
    if gamma1 < 1 or gamma2 < 1:
        raise ValueError("gamma1 and gamma2 must be >= 1")


def _latencies(latency: LatencyModel, context: int, budget: int, draft_budget: Optional[int]):
    latency.check(context, budget)
    db = max(context // 8, 1) if draft_budget is None else draft_budget
    return latency.t_draft(context, db), latency.t_target_retrieval(context, budget), latency.t_target_full(context)


def _inner_round_yield(alpha1: float, gamma1: int) -> np.ndarray:
    """p[y] = probability that one inner round stages y tokens (y = 1..gamma1+1)."""
    p = np.zeros(gamma1 + 2)
    k = np.arange(gamma1)
    p[1:gamma1 + 1] = alpha1 ** k * (1.0 - alpha1)
    p[gamma1 + 1] += alpha1 ** gamma1
    return p


def _inner_phase(alpha1: float, gamma1: int, gamma2: int):
    """Expected inner rounds until >= gamma2 tokens are staged, and the
    distribution of the staged count at that point (a renewal process on the
    partial count 0..gamma2-1, iterated until no mass is left below gamma2)."""
    y = _inner_round_yield(alpha1, gamma1)
    hi = gamma2 + gamma1 + 1
    below = np.zeros(gamma2)          # mass of partial counts still below gamma2
    below[0] = 1.0
    staged = np.zeros(hi)              # mass absorbed at each final count
    rounds = 0.0
    while below.sum() > 1e-15:
        rounds += below.sum()
        nxt = np.zeros(gamma2)
        for s in np.nonzero(below)[0]:
            for inc in np.nonzero(y)[0]:
                t = s + inc
                if t >= gamma2:
                    staged[t] += below[s] * y[inc]
                else:
                    nxt[t] += below[s] * y[inc]
        below = nxt
    return rounds, staged


def hierarchical_speedup(alpha1: float, alpha2: float, gamma1: int, gamma2: int, latency: LatencyModel,
                         context: int, budget: int, draft_budget: Optional[int] = None) -> SpeedupEstimate:
    """Expected tokens and wall time of one outer round of the two-level loop,
    and its speedup over autoregressive decoding on the full cache."""
    _check_rates(alpha1, alpha2, gamma1, gamma2)
    t_d, t_r, t_f = _latencies(latency, context, budget, draft_budget)
    rounds, staged = _inner_phase(alpha1, gamma1, gamma2)
    tokens = float(sum(staged[n] * expected_tokens(alpha2, n) for n in np.nonzero(staged)[0]))
    wall = float(rounds * (gamma1 * t_d + t_r) + t_f)
    return SpeedupEstimate(tokens_per_round=tokens, wall_ms_per_round=wall, speedup=float(tokens * t_f / wall),
                           inner_rounds_per_outer=float(rounds))


def hierarchical_speedup_coarse(alpha1: float, alpha2: float, gamma1: int, gamma2: int, latency: LatencyModel,
                                context: int, budget: int, draft_budget: Optional[int] = None) -> SpeedupEstimate:
    """First-order model: gamma2 / expected_tokens(alpha1, gamma1) inner
    rounds and exactly gamma2 outer proposals (ignores the inner overshoot)."""
    t_d, t_r, t_f = _latencies(latency, context, budget, draft_budget)
    rounds = gamma2 / expected_tokens(alpha1, gamma1)
    tokens = expected_tokens(alpha2, gamma2)
    wall = rounds * (gamma1 * t_d + t_r) + t_f
    return SpeedupEstimate(tokens_per_round=tokens, wall_ms_per_round=wall, speedup=tokens * t_f / wall,
                           inner_rounds_per_outer=rounds)


def _accepted_run(u: np.ndarray, alpha: float, cap) -> np.ndarray:
    """Length of the accepted run before the first rejection, capped at `cap`,
    for i.i.d. acceptances of probability alpha: P(run >= k) = alpha^k, so
    the inverse CDF of one uniform is floor(log u / log alpha)
    (analytics.py:446-457 draws it this way: one uniform per chain)."""
    cap_arr = np.broadcast_to(np.asarray(cap, dtype=np.int64), u.shape)
    if alpha <= 0.0:
        return np.zeros(u.shape, dtype=np.int64)
    if alpha >= 1.0:
        return cap_arr.copy()
    with np.errstate(divide="ignore"):
        run = np.floor(np.log(u) / np.log(alpha))
    run = np.where(np.isfinite(run), run, cap_arr)   # u == 0: the whole cap
    return np.minimum(run.astype(np.int64), cap_arr)


def simulate_speedup(alpha1: float, alpha2: float, gamma1: int, gamma2: int, latency: LatencyModel,
                     context: int, budget: int, rounds: int, seed: int,
                     draft_budget: Optional[int] = None) -> SpeedupEstimate:
    """Monte-Carlo counterpart of hierarchical_speedup (analytics.py:460-499):
    all `rounds` outer rounds advance together, vectorised -- each inner pass
    draws one uniform per round (the accepted draft run, capped at gamma1)
    until every round has staged gamma2 tokens, then one uniform per round
    for the outer run (capped at the staged count).  Same draw order and the
    same 100 batch means for the 95% half-width as the reference, so a seed
    reproduces its estimate."""
    if rounds < 100:
        raise ValueError("need at least 100 simulated rounds")
    _check_rates(alpha1, alpha2, gamma1, gamma2)
    t_d, t_r, t_f = _latencies(latency, context, budget, draft_budget)
    rng = np.random.default_rng(seed)
    staged = np.zeros(rounds, dtype=np.int64)
    inner = np.zeros(rounds, dtype=np.int64)
    pending = np.ones(rounds, dtype=bool)
    while pending.any():
        run = _accepted_run(rng.random(rounds), alpha1, gamma1)   # every round draws, as in the reference
        staged[pending] += run[pending] + 1
        inner[pending] += 1
        pending = staged < gamma2
    tok = _accepted_run(rng.random(rounds), alpha2, staged) + 1
    wall = inner * (gamma1 * t_d + t_r) + t_f
    speed = tok.sum() * t_f / wall.sum()
    nb = 100
    per = rounds // nb
    bt = tok[:nb * per].reshape(nb, per).sum(axis=1).astype(np.float64)
    bw = wall[:nb * per].reshape(nb, per).sum(axis=1)
    bs = bt * t_f / bw
    half = 1.96 * float(bs.std(ddof=1)) / np.sqrt(nb)
    return SpeedupEstimate(tokens_per_round=float(tok.mean()), wall_ms_per_round=float(wall.mean()),
                           speedup=float(speed), ci_halfwidth=half, inner_rounds_per_outer=float(inner.mean()))


# ---------------------------------------------------------------------------
# planted-needle fixtures

@dataclass
class NeedleCase:
    tokens: List[int]
    needle_positions: List[int]
    passkey: bytes
    trigger_position: int


def needle_corpus(context_len: int, n_cases: int, seed: int, passkey_len: int = 6) -> List[NeedleCase]:
    """Byte-token prompts of exactly context_len tokens: BOS, lowercase-letter
    and space filler, a digit passkey starting uniformly inside the middle 80%
    of the context, and a final '?' trigger.  Digits occur only in the
    passkey."""
    if context_len < passkey_len + 8:
        raise ValueError("context too short for a passkey")
    rng = np.random.default_rng(seed)
    alphabet = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz ", dtype=np.uint8).astype(np.int64)
    first = max(1, int(np.ceil(0.1 * context_len)))
    last = int(np.floor(0.9 * context_len)) - passkey_len
    out = []
    for _ in range(n_cases):
        body = alphabet[rng.integers(0, alphabet.size, context_len - 2)].tolist()
        at = int(rng.integers(first, last + 1))
        digits = rng.integers(0, 10, passkey_len)
        key = bytes(int(d) + ord("0") for d in digits)
        toks = [BOS] + body + [ord("?")]
        toks[at:at + passkey_len] = list(key)
        out.append(NeedleCase(tokens=toks, needle_positions=list(range(at, at + passkey_len)), passkey=key,
                              trigger_position=len(toks) - 1))
    return out


def planted_attention_weights(config: ModelConfig, context_len: int, n_needle_tokens: int, strength: float,
                              answer_token: int, seed: int = 0, needle_token_ids: Sequence[int] = DIGIT_TOKENS,
                              designated_layers: Sequence[int] = (0,), margin: float = 2.0) -> ModelWeights:
    """Random weights wired so that, at the designated layers, every decode
    query puts at least `strength` of its attention mass on needle-token
    positions, and attending the needle pushes the output to `answer_token`.

    Construction: two reserved embedding channels -- a query marker carried
    by every token and a key marker carried only by needle tokens -- are
    projected onto the slowest RoPE pair of every head (so relative rotation
    over the context is negligible) with a gain chosen from the required
    softmax logit gap; one value channel carries the key marker through w_o
    into a residual dimension nothing else writes, and only that dimension
    drives the answer logit."""
    if not 0.0 < strength <= 0.99:
        raise ValueError("strength must be in (0, 0.99]")
    if n_needle_tokens < 1 or context_len <= n_needle_tokens:
        raise ValueError("need 1 <= n_needle_tokens < context_len")
    if answer_token in needle_token_ids:
        raise ValueError("answer_token must not be a needle token")
    d, dh = config.d_model, config.head_dim
    if d < 8 or dh < 4:
        raise ValueError("planted construction needs d_model >= 8 and head_dim >= 4")
    slow = dh - 2                                   # even member of the slowest rotation pair
    if 2 * context_len * config.rope_theta ** (-slow / dh) > 0.15:
        raise ValueError(f"rope_theta {config.rope_theta} rotates the slow pair too far over this context; "
                         "use a larger rope_theta")
    w = generate_weights(config, seed, tied_head=False)
    t = w.tensors
    q_ch, k_ch, a_ch = d - 2, d - 1, d - 3          # query marker, key marker, answer channel
    needles = list(needle_token_ids)
    emb = t["embedding"]
    emb[:, q_ch] = 1.0
    emb[:, k_ch] = 0.0
    emb[:, a_ch] = 0.0
    emb[needles, k_ch] = 1.0
    # marker magnitudes after the first RMS norm (its gains start near 1)
    rms = np.sqrt(np.mean(emb.astype(np.float64) ** 2, axis=1) + config.norm_eps)
    qn = float(np.min(1.0 / rms))
    kn = float(np.min(emb[needles, k_ch].astype(np.float64) / rms[needles]))
    # logit gap so that n needles out of context_len keys hold `strength` of the mass, plus a margin
    gap = np.log(strength / (1.0 - strength) * (context_len - n_needle_tokens) / n_needle_tokens) + margin
    gain = float(np.sqrt(max(gap, 1.0) * np.sqrt(dh) / (qn * kn)))
    for li in designated_layers:
        wq, wk = t[f"layers.{li}.wq"], t[f"layers.{li}.wk"]
        wq[q_ch, :] = 0.0
        wk[k_ch, :] = 0.0
        wq[q_ch, slow::dh] = gain                   # column h*dh + slow of every query head
        wk[k_ch, slow::dh] = gain                   # ... and of every kv head
    li = designated_layers[0]
    wv, wo = t[f"layers.{li}.wv"], t[f"layers.{li}.wo"]
    wv[:, 0] = 0.0
    wv[k_ch, 0] = 1.0                               # value dim 0 of kv head 0 = the key marker
    wo[:, a_ch] = 0.0
    wo[0, a_ch] = 1.0                               # attention channel 0 -> answer channel only
    head = t["lm_head"]
    head[a_ch, :] = 0.0
    head[a_ch, answer_token] = 1.0
    return ModelWeights(config, t, False).validate()
