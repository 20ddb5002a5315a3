"""World-size-2 protocol test of the sequence-sharded full cache on CPU
(gloo): the shard plan, the rank-ordered partial-softmax merge and the
global chunk selection from per-shard scores, exchanged over real
torch.distributed collectives, equal the unsharded oracle results.  The GPU
path runs the same protocol over NCCL inside libhs_b200 (hs_forward with an
HsShard, RetrievalCache._score); tests/test_gpu_shard.py checks its kernels."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import hs_oracle as O
    from paper_2404_11912_b200.shard import shard_chunk_counts, shard_plan

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        for case, (n, t, chunk, budget) in enumerate(((1203, 5, 8, 128), (64, 1, 4, 16), (999, 7, 16, 256))):
            rng = np.random.default_rng(case)      # same data on every rank
            dh, H = 16, 4
            K = O.bf16_round(rng.normal(0, 1, (n, dh)).astype(np.float32))
            V = O.bf16_round(rng.normal(0, 1, (n, dh)).astype(np.float32))
            q = rng.normal(0, 1, (t, dh)).astype(np.float32)
            plan = shard_plan(n, world, chunk)
            lo, hi = plan[rank]
            end = n if hi is None else min(n, hi)
            assert lo % chunk == 0
            # ---- attention: this rank's partial state, all-gathered, merged in rank order
            (m, l, o), = O.shard_partials(q, K, V, [lo, max(lo, end)] if end > lo else [0, 0], 1 / np.sqrt(dh))
            if end <= lo:
                m, l, o = np.full(t, -np.inf), np.zeros(t), np.zeros((t, dh))
            packed = torch.from_numpy(np.concatenate([m[:, None], l[:, None], o], axis=1))
            got = [torch.empty_like(packed) for _ in range(world)]
            dist.all_gather(got, packed)
            parts = [(g[:, 0].numpy(), g[:, 1].numpy(), g[:, 2:].numpy()) for g in got]
            merged = O.merge_partials(parts)
            whole = O.merge_partials(O.shard_partials(q, K, V, [0, n], 1 / np.sqrt(dh)))
            assert np.allclose(merged, whole, rtol=1e-12, atol=1e-12)
            # ---- build: per-shard chunk scores -> all-gather -> replicated selection
            keys = O.bf16_round(rng.normal(0, 1, (n, 2, dh)).astype(np.float32))
            qh = rng.normal(0, 1, (H, dh)).astype(np.float32)
            counts = shard_chunk_counts(plan, n, chunk)
            cmax = max(counts)
            mine = np.zeros(cmax)
            if counts[rank]:
                _, sc = O.chunk_scores(keys[lo:end], qh, chunk, 2)
                mine[:counts[rank]] = sc
            allsc = [torch.empty(cmax, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(allsc, torch.from_numpy(mine))
            scores = np.concatenate([allsc[r].numpy()[:counts[r]] for r in range(world)])
            _, ref = O.chunk_scores(keys, qh, chunk, 2)
            assert np.array_equal(scores, ref)
            quota = budget // chunk
            assert O.select_chunks(scores, quota, budget >= n) == O.select_chunks(ref, quota, budget >= n)
    finally:
        dist.destroy_process_group()


def test_shard_plan_is_chunk_aligned_and_covers_the_context():
    from paper_2404_11912_b200.shard import shard_chunk_counts, shard_plan
    for n, world, chunk in ((122880, 8, 8), (1048576, 8, 16), (100, 3, 8), (5, 4, 1), (7, 1, 32)):
        plan = shard_plan(n, world, chunk)
        assert len(plan) == world and plan[0][0] == 0 and plan[-1][1] is None
        for (lo, hi), (lo2, _) in zip(plan[:-1], plan[1:]):
            assert hi == lo2 and lo % chunk == 0 and hi % chunk == 0
        counts = shard_chunk_counts(plan, n, chunk)
        assert sum(counts) == -(-n // chunk)


def test_world2_gloo_protocol_matches_unsharded():
    port = _free_port()
    mp.spawn(_worker, args=(2, port), nprocs=2, join=True)


def test_shard_plan_properties():
    """Property check over random geometries (hypothesis): every position has
    exactly one owner, boundaries are chunk-aligned, no retrieval chunk
    straddles two ranks, and the per-rank chunk counts add up."""
    hyp = pytest.importorskip("hypothesis")
    st = hyp.strategies
    from paper_2404_11912_b200.shard import shard_chunk_counts, shard_plan

    @hyp.settings(max_examples=200, deadline=None)
    @hyp.given(n=st.integers(1, 1 << 21), world=st.integers(1, 8), chunk=st.sampled_from([1, 4, 8, 16, 32]),
               probe=st.integers(0, (1 << 21) + 4096))
    def check(n, world, chunk, probe):
        plan = shard_plan(n, world, chunk)
        owners = [r for r, (lo, hi) in enumerate(plan) if lo <= probe and (hi is None or probe < hi)]
        assert len(owners) == 1
        r = owners[0]
        lo, hi = plan[r]
        c0 = probe // chunk * chunk                       # the probe's chunk lies on the same rank
        assert lo <= c0 and (hi is None or c0 + chunk <= hi)
        assert all(b % chunk == 0 for lo_, hi_ in plan for b in (lo_, hi_) if b is not None)
        assert sum(shard_chunk_counts(plan, n, chunk)) == -(-n // chunk)

    check()
