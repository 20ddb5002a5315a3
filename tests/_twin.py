"""Test infrastructure: a CPU-oracle twin of a GPU HierarchicalSession.

`oracle_twin` copies the GPU session's complete state -- full cache K/V,
StreamingLLM draft cache, the built retrieval cache (selected entries in
position order, victim FIFO, positions) and every lane's frontier logits row
-- into an `oracle.hs_oracle.OSession`, so the GPU and the CPU oracle then
run the same Algorithm-1 rounds from IDENTICAL inputs (the north star's
parity setting).  Values are copied exactly (bf16 cache entries as fp64 /
fp32, logits rows as fp32).
"""

from __future__ import annotations

import numpy as np
import torch


def _rows_from(O, K, V, pos, f64=False):
    r = O._Rows(K.shape[1], K.shape[2], cap=max(16, K.shape[0] + 256), dtype=np.float64 if f64 else np.float32)
    if K.shape[0]:
        r.add(K, V, pos)
    return r


def oracle_twin(O, s, om, odm, ospec):
    """OSession holding exactly the state of GPU session `s` (unsharded)."""
    o = object.__new__(O.OSession)
    o.spec, o.committed = ospec, list(s.committed)
    fc, sc, rc = s.full_lane.cache, s.draft_lane.cache, s.retr_lane.cache
    tc, dc = om.cfg, odm.cfg
    # full cache: positions [0, frontier), slot == position
    n = fc.frontier
    full = O.OFullCache(tc.n_layers, tc.n_kv_heads, tc.head_dim, tc.max_seq, kv_bf16=True)
    full.rows = [_rows_from(O, fc.k[l, :, :n].permute(1, 0, 2).float().cpu().numpy(),
                            fc.v[l, :, :n].permute(1, 0, 2).float().cpu().numpy(), np.arange(n), f64=True)
                 for l in range(tc.n_layers)]
    full.frontier, full.committed = fc.frontier, fc.committed
    # draft StreamingLLM cache: the stored positions (sinks + window) in position order
    st = O.OStreamingCache(dc.n_layers, dc.n_kv_heads, dc.head_dim, sc.config.n_sink, sc.config.budget, kv_bf16=True)
    keep = sc._store(sc.frontier)
    slots = torch.as_tensor([sc._slot(int(p)) for p in keep], dtype=torch.long, device=sc.k.device)
    st.rows = [_rows_from(O, sc.k[l][:, slots].permute(1, 0, 2).float().cpu().numpy(),
                          sc.v[l][:, slots].permute(1, 0, 2).float().cpu().numpy(), keep.astype(np.int64))
               for l in range(dc.n_layers)]
    st.frontier, st.committed = sc.frontier, sc.committed
    # retrieval cache right after a build: selection in position order, empty tail
    if rc.frontier != rc.committed:
        raise ValueError("twin needs a retrieval cache without a speculative tail")
    rt = O.ORetrievalCache(tc.n_layers, tc.n_kv_heads, tc.head_dim, rc.config.chunk_size, rc.config.budget,
                           kv_bf16=True)
    for l in range(tc.n_layers):
        pos = rc.pos[l, :rc.n_sel].cpu().numpy().astype(np.int64)
        order = np.argsort(pos, kind="stable")
        idx = torch.as_tensor(order, device=rc.k.device)
        K = rc.k[l][:, :rc.n_sel].index_select(1, idx).permute(1, 0, 2).float().cpu().numpy()
        V = rc.v[l][:, :rc.n_sel].index_select(1, idx).permute(1, 0, 2).float().cpu().numpy()
        rt.sel[l] = _rows_from(O, K, V, pos[order])
        ring = rc.ring[l, :rc.n_sel].cpu().numpy()
        head = rc.ring_head
        rt.victims[l] = [int(pos[ring[(head + i) % rc.n_sel]]) for i in range(rc.n_sel)]
    rt.frontier, rt.committed = rc.frontier, rc.committed
    o.full, o.draft, o.retr = O.OLane(om, full), O.OLane(odm, st), O.OLane(om, rt)
    for ol, gl in ((o.full, s.full_lane), (o.draft, s.draft_lane), (o.retr, s.retr_lane)):
        ol.row = gl._front.cpu().numpy().copy() if gl._has_front else None
    o.builds = []
    o.rolling = O.ORolling(ospec.rolling_window)
    o.rolling.rates = list(s.rolling.rates)
    o.since_build = s.tokens_since_build
    return o
