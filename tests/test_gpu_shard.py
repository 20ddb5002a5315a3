"""Sequence-sharded full cache on one B200 (`-m gpu`).

The driver's GPU boxes have one GPU, so the multi-rank exchange is checked
in two halves: (1) the NCCL code path itself runs with a one-rank
communicator and must reproduce the unsharded path bit for bit; (2) the
math of G shards -- per-shard partial states merged in rank order, per-shard
chunk scores, zero-padded per-shard gathers summed -- runs on one device and
must equal the unsharded results.  The world-size-2 protocol over real
collectives is covered on CPU with gloo (tests/test_shard_cpu.py)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2404_11912_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def one_rank(P):
    from paper_2404_11912_b200.shard import SequenceShards
    sh = SequenceShards.single()
    yield sh
    sh.destroy()


def _planted(P, seed=5):
    tc = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=128, d_ff=344, vocab_size=512, max_seq=2048)
    dc = P.ModelConfig(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=64, d_ff=172, vocab_size=512, max_seq=2048)
    tw = P.plant_successor(P.generate_weights(tc, seed, tied_head=False), 9, 0.9)
    dw = P.plant_successor(P.generate_weights(dc, seed + 1, tied_head=False), 9, 0.9)
    return tw, dw


def test_one_rank_sharded_forward_is_bitwise_unsharded(P, one_rank):
    tw, _ = _planted(P)
    prompt = np.random.default_rng(0).integers(1, 512, 700).tolist()
    a = P.FullCache.from_config(tw.config)
    b = P.FullCache.shard(tw.config, one_rank, len(prompt), 8)
    # the row-exact decode path on both sides (the GEMM prefill is unsharded-only)
    from paper_2404_11912_b200 import model as M
    la = M._host_rows(M.forward_device(tw, prompt, a, None, prefill=False))
    lb = M._host_rows(M.forward_device(tw, prompt, b, None, prefill=False))
    a.commit(a.frontier)
    b.commit(b.frontier)
    assert np.array_equal(la, lb)
    for tok in (3, 17, 400):
        assert np.array_equal(P.decode_step(tw, tok, a), P.decode_step(tw, tok, b))
    assert np.array_equal(P.decode_chunk(tw, [5, 6, 7, 8, 9], a), P.decode_chunk(tw, [5, 6, 7, 8, 9], b))


def test_one_rank_sharded_session_matches_unsharded(P, one_rank):
    tw, dw = _planted(P)
    prompt = np.random.default_rng(1).integers(1, 512, 900).tolist()
    spec = P.SpecConfig(target_len=900 + 80, gamma1=2, gamma2=4, temperature=0.6, seed=3,
                        streaming=P.StreamingConfig(n_sink=4, budget=128),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=128, rebuild_stride=24))
    from paper_2404_11912_b200 import model as M
    keep = M.PREFILL_MIN_ROWS
    M.PREFILL_MIN_ROWS = 10 ** 9      # unsharded prompt through the row-exact path too: bitwise comparison
    try:
        out_a, tr_a = P.HierarchicalSession(tw, dw, prompt, spec).generate()
        out_b, tr_b = P.HierarchicalSession(tw, dw, prompt, spec, shards=one_rank).generate()
        assert out_a == out_b
        assert tr_a.summary() == tr_b.summary()
        ar = P.autoregressive_generate(tw, prompt, 900 + 20, 0.0, 0, shards=one_rank, chunk=8)
        assert ar == P.autoregressive_generate(tw, prompt, 900 + 20, 0.0, 0)
    finally:
        M.PREFILL_MIN_ROWS = keep


def _fill(cache, K, V, positions):
    """write rows at absolute positions into a (possibly sharded) full cache"""
    for l in range(cache.n_layers):
        cache._n[l] = 0
        cache.append(l, K[l], V[l])
    cache.frontier = cache.committed = len(positions)


def test_shard_partials_merge_equals_unsharded_attention(P):
    """G shard caches over one sequence: hs_attention_partial per shard +
    hs_shard_merge (rank order) == hs_attention over the whole cache."""
    from paper_2404_11912_b200._abi import HsStep, check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr, workspaces
    from paper_2404_11912_b200.shard import shard_plan
    rng = np.random.default_rng(7)
    L, kvh, H, dh = 1, 4, 8, 128
    for n, G, t, dh in ((6000, 4, 7, 128), (5000, 3, 1, 128), (777, 2, 5, 64), (333, 4, 3, 64)):
        K = rng.normal(0, 1, (L, n, kvh, dh)).astype(np.float32)
        V = rng.normal(0, 1, (L, n, kvh, dh)).astype(np.float32)
        q = torch.from_numpy(rng.normal(0, 1, (t, H, dh)).astype(np.float32)).cuda()
        full = P.FullCache(L, kvh, dh, n + 64)
        _fill(full, K, V, range(n))
        st = HsStep()
        st.pos0, st.n_view, st.split = n - t, n, 1024
        nb = lib.hs_attention_workspace_bytes(t, H, dh, n, 1024)
        ws = workspaces.get("shard_t", nb)
        ref = torch.zeros((t, H * dh), device="cuda")
        check(lib.hs_attention(full._ref, 0, C.byref(st), H, ptr(q), t, ptr(ref), ptr(ws), nb, stream_ptr()))
        parts = torch.zeros((G, t * H, dh + 2), device="cuda")
        for r, (lo, hi) in enumerate(shard_plan(n, G, 8)):
            sc = P.FullCache(L, kvh, dh, n + 64, None, lo, hi)
            end = n if hi is None else min(n, hi)
            if end > lo:
                for l in range(L):
                    sc._write_rows(l, K[l, lo:end], V[l, lo:end], np.arange(end - lo), np.arange(lo, end))
            s2 = HsStep()
            s2.pos0, s2.n_view, s2.split, s2.pos_base = n - t, max(0, end - lo), 1024, lo
            check(lib.hs_attention_partial(sc._ref, 0, C.byref(s2), H, ptr(q), t, ptr(parts[r]), ptr(ws), nb,
                                           stream_ptr()))
        out = torch.zeros((t, H * dh), device="cuda")
        check(lib.hs_shard_merge(ptr(parts), G, t * H, dh, ptr(out), stream_ptr()))
        a, b = out.cpu().numpy(), ref.cpu().numpy()
        assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max(), (n, G, t)


def test_shard_scores_and_gathers_assemble_the_unsharded_build(P):
    """Per-shard chunk scores concatenated in rank order are bit-identical to
    the unsharded scores; per-shard gathers (foreign chunks left untouched,
    here zero-initialised) sum to the unsharded retrieval buffer."""
    from paper_2404_11912_b200._abi import check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr
    from paper_2404_11912_b200.shard import shard_chunk_counts, shard_plan
    rng = np.random.default_rng(11)
    L, kvh, H, dh, chunk, budget = 2, 2, 4, 64, 8, 256
    for n, G in ((3001, 2), (4096, 4), (999, 3)):
        K = rng.normal(0, 1, (L, n, kvh, dh)).astype(np.float32)
        V = rng.normal(0, 1, (L, n, kvh, dh)).astype(np.float32)
        q = rng.normal(0, 1, (L, H, dh)).astype(np.float32)
        full = P.FullCache(L, kvh, dh, n + 64)
        _fill(full, K, V, range(n))
        rc = P.RetrievalCache(L, kvh, dh, P.RetrievalConfig(chunk_size=chunk, budget=budget))
        table = rc.build(full, q, n)
        want_scores = np.stack(table.scores)
        plan = shard_plan(n, G, chunk)
        counts = shard_chunk_counts(plan, n, chunk)
        qd = torch.from_numpy(q).cuda()
        got, acc_k, acc_v = [], torch.zeros_like(rc.k, dtype=torch.float32), torch.zeros_like(rc.v, dtype=torch.float32)
        for r, (lo, hi) in enumerate(plan):
            sc = P.FullCache(L, kvh, dh, n + 64, None, lo, hi)
            end = n if hi is None else min(n, hi)
            for l in range(L):
                if end > lo:
                    sc._write_rows(l, K[l, lo:end], V[l, lo:end], np.arange(end - lo), np.arange(lo, end))
            out = torch.empty((L, counts[r]), dtype=torch.float64, device="cuda")
            if counts[r]:
                check(lib.hs_chunk_score(ptr(sc.k), 1, kvh * sc.cap * dh, sc.cap * dh, dh, L, kvh, dh, end - lo,
                                         chunk, ptr(qd), H, ptr(out), stream_ptr()))
            got.append(out.cpu().numpy())
            part = P.RetrievalCache(L, kvh, dh, P.RetrievalConfig(chunk_size=chunk, budget=budget))
            part.chosen.copy_(rc.chosen)
            nch = int(rc.table._n_imp)
            check(lib.hs_retrieval_gather(sc._ref, part._ref, ptr(part.chosen), part.quota, nch, chunk, n, lo,
                                          hi or 0, stream_ptr()))
            acc_k += part.k.float()
            acc_v += part.v.float()
            assert torch.equal(part.pos[:, :rc.n_sel], rc.pos[:, :rc.n_sel])
        assert np.array_equal(np.concatenate(got, axis=1), want_scores)
        assert torch.equal(acc_k[:, :, :rc.n_sel].to(torch.bfloat16), rc.k[:, :, :rc.n_sel])
        assert torch.equal(acc_v[:, :, :rc.n_sel].to(torch.bfloat16), rc.v[:, :, :rc.n_sel])


def test_sharded_cache_rejects_misaligned_bounds(P):
    from paper_2404_11912_b200._abi import check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr
    src = P.FullCache(1, 2, 64, 512, None, 4, 260)
    dst = P.RetrievalCache(1, 2, 64, P.RetrievalConfig(chunk_size=8, budget=64))
    with pytest.raises(ValueError):
        check(lib.hs_retrieval_gather(src._ref, dst._ref, ptr(dst.chosen), dst.quota, 1, 8, 100, 4, 260,
                                      stream_ptr()))


def _causal_ref(q, K, V, pos0, positions):
    """fp64 causal attention: q [t][H][dh] at positions pos0.., keys K/V [n][KVH][dh]
    at `positions` (model.py:290-315 with the prefix mask)."""
    t, H, dh = q.shape
    KVH = K.shape[1]
    g = H // KVH
    out = np.zeros((t, H, dh))
    for i in range(t):
        vis = positions <= pos0 + i
        for h in range(H):
            k, v = K[vis, h // g].astype(np.float64), V[vis, h // g].astype(np.float64)
            s = k @ q[i, h].astype(np.float64) / np.sqrt(dh)
            w = np.exp(s - s.max())
            out[i, h] = w @ v / w.sum()
    return out


def test_prefill_attention_kernel_and_shard_merge(P):
    """The 128-row tensor-core prefill attention (hs_prefill_attention)
    against fp64 causal attention, and its per-shard partial states merged in
    rank order (hs_shard_merge) against the unsharded kernel output."""
    from paper_2404_11912_b200._abi import HsStep, check, lib
    from paper_2404_11912_b200.runtime import ptr, stream_ptr
    from paper_2404_11912_b200.shard import shard_plan
    rng = np.random.default_rng(21)
    L, kvh, H, dh = 1, 2, 4, 128
    for n, t, G in ((700, 300, 3), (1500, 1500, 2), (2100, 129, 4)):
        pos0 = n - t
        K = rng.normal(0, 1, (L, n, kvh, dh)).astype(np.float32)
        V = rng.normal(0, 1, (L, n, kvh, dh)).astype(np.float32)
        qh = rng.normal(0, 1, (t, H, dh)).astype(np.float32)
        q = torch.from_numpy(qh).cuda()
        full = P.FullCache(L, kvh, dh, n + 64)
        _fill(full, K, V, range(n))
        st = HsStep()
        st.pos0, st.n_view = pos0, n
        out = torch.zeros((t, H * dh), device="cuda")
        check(lib.hs_prefill_attention(full._ref, 0, C.byref(st), H, ptr(q), t, ptr(out), None, stream_ptr()))
        Kb = full.k[0, :, :n].float().permute(1, 0, 2).cpu().numpy()    # bf16-stored keys as the kernel sees them
        Vb = full.v[0, :, :n].float().permute(1, 0, 2).cpu().numpy()
        ref = _causal_ref(qh, Kb, Vb, pos0, np.arange(n)).reshape(t, H * dh)
        got = out.cpu().numpy()
        assert np.abs(got - ref).max() <= 3e-5 * np.abs(ref).max(), (n, t)
        parts = torch.zeros((G, t * H, dh + 2), device="cuda")
        for r, (lo, hi) in enumerate(shard_plan(n, G, 8)):
            sc = P.FullCache(L, kvh, dh, n + 64, None, lo, hi)
            end = n if hi is None else min(n, hi)
            if end > lo:
                sc._write_rows(0, K[0, lo:end], V[0, lo:end], np.arange(end - lo), np.arange(lo, end))
            s2 = HsStep()
            s2.pos0, s2.n_view, s2.pos_base = pos0, max(0, end - lo), lo
            check(lib.hs_prefill_attention(sc._ref, 0, C.byref(s2), H, ptr(q), t, None, ptr(parts[r]), stream_ptr()))
        merged = torch.zeros((t, H * dh), device="cuda")
        check(lib.hs_shard_merge(ptr(parts), G, t * H, dh, ptr(merged), stream_ptr()))
        assert np.abs(merged.cpu().numpy() - got).max() <= 1e-5 * np.abs(got).max(), (n, t, G)


def test_one_rank_sharded_prefill_matches_unsharded(P, one_rank):
    """hs_prefill_sharded through a one-rank NCCL communicator (partial states,
    all-gather, merge) against the unsharded GEMM prefill, and the decode that
    follows."""
    cfg = P.ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=128, d_ff=344, vocab_size=512, max_seq=2048)
    w = P.generate_weights(cfg, 9, tied_head=False)
    prompt = np.random.default_rng(4).integers(1, 512, 900).tolist()
    a = P.FullCache.from_config(cfg)
    b = P.FullCache.shard(cfg, one_rank, len(prompt), 8)
    la, lb = P.prefill(w, prompt, a), P.prefill(w, prompt, b)
    assert np.allclose(la, lb, rtol=1e-5, atol=1e-5 * np.abs(la).max())
    assert (np.argmax(la, -1) == np.argmax(lb, -1)).mean() > 0.999
    da, db = P.decode_step(w, 17, a), P.decode_step(w, 17, b)
    assert np.allclose(da, db, rtol=1e-4, atol=1e-4 * np.abs(da).max())


def _run_ranks(fn, world, shards=None):
    """Run fn(rank) on `world` host threads, each with its own CUDA stream
    (the loopback group's execution model); a failing rank aborts the group
    so its peers fail fast; re-raise the first failure."""
    import threading
    out, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:   # noqa: BLE001 - re-raised below
            errs.append((r, e))
            if shards is not None:
                shards[r].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0][1]
    return out


@pytest.mark.parametrize("G", [2, 4, 8])
def test_loopback_shards_session_matches_unsharded(P, G):
    """G sequence shards on ONE GPU through the loopback group (G host
    threads and streams; all-gather / all-gather-v as device copies with the
    NCCL calls' semantics) run the whole sharded product path: sharded GEMM
    prefill, per-layer partial-state exchange in every full-cache forward,
    sharded rebuilds (per-shard scores + the chunk exchange) and the decoded
    tail appended to the last shard.  Every rank's session equals the
    unsharded one: token stream, per-level counts, rebuilds and the
    retrieval cache's positions exactly; logits and the cached K/V to fp32
    accumulation noise (the G per-shard partial softmax states merge in a
    different order than one GPU's splits)."""
    from paper_2404_11912_b200.shard import SequenceShards
    tw, dw = _planted(P, seed=7)
    tw.device(), dw.device()                 # pack once, before the threads share them
    prompt = np.random.default_rng(2).integers(1, 512, 900).tolist()
    spec = P.SpecConfig(target_len=900 + 96, gamma1=2, gamma2=4, temperature=0.6, seed=5,
                        streaming=P.StreamingConfig(n_sink=4, budget=128),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=128, rebuild_stride=24))
    ref = P.HierarchicalSession(tw, dw, prompt, spec)
    ref_out, ref_tr = ref.generate()
    shards = SequenceShards.loopback(G)

    def rank(r):
        s = P.HierarchicalSession(tw, dw, prompt, spec, shards=shards[r])
        out, tr = s.generate()
        fc = s.full_lane.cache
        lo, n = fc.lo, fc._local(fc.frontier)
        return (out, tr.summary(), s.rebuilds, s.retr_lane.cache.pos.clone(), lo, n,
                fc.k[:, :, :n].clone(), s.full_lane._front.clone())

    try:
        res = _run_ranks(rank, G, shards)
    finally:
        shards[0].destroy()
    for r, (out, summ, rebuilds, rpos, lo, n, k, front) in enumerate(res):
        assert out == ref_out, r
        assert summ == ref_tr.summary(), r
        assert rebuilds == ref.rebuilds and rebuilds >= 2, (r, rebuilds)
        assert torch.equal(rpos, ref.retr_lane.cache.pos), r
        # this rank's slice of the full cache (the last rank holds the decoded tail)
        want = ref.full_lane.cache.k[:, :, lo:lo + n].float()
        assert torch.allclose(k.float(), want, rtol=2 ** -7, atol=1e-6), r
        f0 = ref.full_lane._front
        assert (front - f0).abs().max().item() <= 1e-5 * f0.abs().max().item(), r
    assert res[-1][5] > 0 and res[-1][4] + res[-1][5] == ref.full_lane.cache.frontier


def test_loopback_collectives(P):
    """all_gather / all_gather_v / sum all_reduce over a 3-rank loopback group
    equal their definitions (rank order)."""
    from paper_2404_11912_b200.shard import SequenceShards
    G = 3
    shards = SequenceShards.loopback(G)
    try:
        def rank(r):
            sh = shards[r]
            x = torch.arange(5, dtype=torch.float64, device="cuda") + 10 * r
            g = sh.all_gather(x)
            v = sh.all_gather_v(torch.full((r + 1,), float(r), device="cuda"), [1, 2, 3])
            y = torch.full((7,), 0.5 * (r + 1), dtype=torch.float32, device="cuda")
            sh.all_reduce_sum_(y)
            b = torch.full((4,), 1.0 + r, dtype=torch.bfloat16, device="cuda")
            sh.all_reduce_sum_(b)
            sh.check()
            return g.cpu(), v.cpu(), y.cpu(), b.float().cpu()

        for g, v, y, b in _run_ranks(rank, G, shards):
            assert torch.equal(g, torch.stack([torch.arange(5, dtype=torch.float64) + 10 * r for r in range(G)]))
            assert torch.equal(v, torch.tensor([0.0, 1, 1, 2, 2, 2]))
            assert torch.equal(y, torch.full((7,), 3.0))
            assert torch.equal(b, torch.full((4,), 6.0))
    finally:
        shards[0].destroy()


# ---------------------------------------------------------------------------
# tensor-parallel dense layers (hs_forward_tp)

def test_one_rank_tensor_parallel_is_bitwise_replicated(P, one_rank):
    """World 1 through the NCCL code path: the row block is the whole matrix
    (same K split), the all-gather a copy and norm_prep rebuilds the operand
    the GEMV epilogue would have written -- logits bitwise equal to hs_forward,
    for decode steps, verify blocks and a whole session (TP on the full and
    retrieval lanes)."""
    from paper_2404_11912_b200 import model as M
    tw, dw = _planted(P)
    prompt = np.random.default_rng(0).integers(1, 512, 600).tolist()
    a = P.FullCache.from_config(tw.config)
    b = P.FullCache.from_config(tw.config)
    P.prefill(tw, prompt, a)
    P.prefill(tw, prompt, b)
    for toks in ([3], [17, 18, 19, 20, 21], [7] * 8):
        la = M._host_rows(M.forward_device(tw, toks, a))
        lb = M._host_rows(M.forward_device(tw, toks, b, tp=one_rank))
        assert np.array_equal(la, lb), len(toks)
    spec = P.SpecConfig(target_len=600 + 64, gamma1=2, gamma2=4, temperature=0.6, seed=3,
                        streaming=P.StreamingConfig(n_sink=4, budget=128),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=128, rebuild_stride=24))
    sa = P.HierarchicalSession(tw, dw, prompt, spec)
    sb = P.HierarchicalSession(tw, dw, prompt, spec, tp=one_rank)   # (the sharded GEMM prefill is not bitwise)
    out_a, tr_a = sa.generate()
    out_b, tr_b = sb.generate()
    assert out_a == out_b and tr_a.summary() == tr_b.summary()
    assert torch.equal(sa.full_lane._front, sb.full_lane._front)
    with pytest.raises(ValueError):    # probes / batches > 8 rows are not tensor-parallel
        from paper_2404_11912_b200._abi import check, lib
        from paper_2404_11912_b200.runtime import ptr, stream_ptr
        dm = tw.device()
        st = b._step(9)
        nb = lib.hs_forward_tp_workspace_bytes(dm.ref, 9, st.n_view, st.split, 0, 1)
        ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        tok = torch.ones(9, dtype=torch.int32, device="cuda")
        out = torch.empty((9, tw.config.vocab_size), device="cuda")
        check(lib.hs_forward_tp(dm.ref, b._ref, C.byref(st), None, one_rank.ref, ptr(tok), 9, ptr(out), None,
                                ptr(ws), nb, stream_ptr()))


@pytest.mark.parametrize("G,seq", [(2, True), (4, True), (8, True), (3, False)])
def test_loopback_tensor_parallel_session(P, G, seq):
    """G ranks on one GPU (loopback group): every projection of the target's
    full and retrieval lanes split by output rows over the ranks (rank r
    streams 1/G of the weight bytes; with 8 ranks several own no tile of the
    small test matrices), optionally with the full cache also sequence-
    sharded.  Every rank ends bitwise identical to the others; against one
    GPU the K splits of the smaller row blocks differ, so logits agree to
    fp32 accumulation noise and the greedy stream and counts are equal."""
    from paper_2404_11912_b200.shard import SequenceShards
    tw, dw = _planted(P, seed=7)
    tw.device(), dw.device()
    prompt = np.random.default_rng(2).integers(1, 512, 700).tolist()
    spec = P.SpecConfig(target_len=700 + 72, gamma1=2, gamma2=4, temperature=0.0, seed=5,
                        streaming=P.StreamingConfig(n_sink=4, budget=128),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=128, rebuild_stride=24))
    ref = P.HierarchicalSession(tw, dw, prompt, spec)
    ref_out, ref_tr = ref.generate()
    shards = SequenceShards.loopback(G)

    def rank(r):
        s = P.HierarchicalSession(tw, dw, prompt, spec, shards=shards[r] if seq else None, tp=shards[r])
        out, tr = s.generate()
        return out, tr.summary(), s.full_lane._front.clone(), s.retr_lane._front.clone()

    try:
        res = _run_ranks(rank, G, shards)
    finally:
        shards[0].destroy()
    f0 = ref.full_lane._front
    for r, (out, summ, front, rfront) in enumerate(res):
        assert out == ref_out, r
        assert summ == ref_tr.summary(), r
        assert torch.equal(front, res[0][2]) and torch.equal(rfront, res[0][3]), r
        assert (front - f0).abs().max().item() <= 1e-5 * f0.abs().max().item(), r
