"""Per-round trace of config 1 at T=0.6 on the GPU package (or the oracle with --oracle)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import hs_oracle as O

def cfgs():
    t = dict(n_layers=2, n_heads=4, n_kv_heads=4, head_dim=64, d_ff=688, vocab_size=260, max_seq=4224)
    d = dict(n_layers=1, n_heads=2, n_kv_heads=2, head_dim=64, d_ff=344, vocab_size=260, max_seq=4224)
    return t, d

prompt = np.random.default_rng(0).integers(1, 256, 4096).tolist()
T = float(sys.argv[2]) if len(sys.argv) > 2 else 0.6
if sys.argv[1] == "oracle":
    t, d = cfgs()
    tm = O.OModel(O.OConfig(**t), O.round_weights_bf16(O.make_tensors(O.OConfig(**t), 1, False)), False)
    dm = O.OModel(O.OConfig(**d), O.round_weights_bf16(O.make_tensors(O.OConfig(**d), 2, False)), False)
    s = O.OSession(tm, dm, prompt, O.OSpec(target_len=4160, gamma1=2, gamma2=4, temperature=T, seed=0, n_sink=4,
                   stream_budget=256, chunk=8, retr_budget=256), kv_bf16=True)
    rng = np.random.default_rng(0); tr = O.OTrace(); rounds = []
    while len(s.committed) < 4160:
        nb = len(s.builds); n0 = len(s.committed)
        s.round(rng, tr)
        rounds.append([n0, len(s.committed) - n0, len(s.builds) - nb, tr.inner[1], tr.outer[1]])
    print(json.dumps({"tokens": s.committed[4096:], "rounds": rounds,
                      "imp": [[list(map(int, b[0][l][2])) for l in range(2)] for b in s.builds]}))
else:
    import paper_2404_11912_b200 as P
    from paper_2404_11912_b200 import speculation as S
    t, d = cfgs()
    def bw(w):
        return P.ModelWeights(w.config, O.round_weights_bf16(w.tensors), w.tied_head)
    tw = bw(P.generate_weights(P.ModelConfig(**t), 1, tied_head=False))
    dw = bw(P.generate_weights(P.ModelConfig(**d), 2, tied_head=False))
    spec = P.SpecConfig(target_len=4160, gamma1=2, gamma2=4, temperature=T, seed=0,
                        streaming=P.StreamingConfig(n_sink=4, budget=256),
                        retrieval=P.RetrievalConfig(chunk_size=8, budget=256))
    s = P.HierarchicalSession(tw, dw, prompt, spec)
    imps = [s.retr_lane.cache.table.selected]
    orig = s._maybe_rebuild
    def mr():
        r = orig()
        if r: imps.append(s.retr_lane.cache.table.selected)
        return r
    s._maybe_rebuild = mr
    out, tr = s.generate()
    print(json.dumps({"tokens": out[4096:], "summary": tr.summary(), "imp": imps,
                      "rounds": [r["outer_round"] for r in tr.records]}))
