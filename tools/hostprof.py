import cProfile, pstats, sys, os
sys.path.insert(0, '/root/repo')
os.chdir('/root/repo')
import numpy as np, torch
import bench, paper_2404_11912_b200 as P
tdm, ddm = P.DeviceModel.random(P.ModelConfig(**bench.TARGET_7B), seed=1), P.DeviceModel.random(P.ModelConfig(**bench.DRAFT_68M), seed=1001)
tdm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC); ddm.plant_successor_(bench.PLANT_SEED, bench.EASY_FRAC)
tw, dw = P.ModelWeights.on_device(tdm), P.ModelWeights.on_device(ddm)
ctx = np.random.default_rng(0).integers(1, 32000, 32768).tolist()
spec = P.SpecConfig(target_len=32769, gamma1=2, gamma2=4, streaming=P.StreamingConfig(n_sink=4, budget=256), retrieval=P.RetrievalConfig(chunk_size=8, budget=4096))
sess = P.HierarchicalSession.synthetic(tw, dw, ctx, spec)
for i in range(2):
    sess.config.target_len = len(sess.committed) + 16; sess.generate(seed=i)
torch.cuda.synchronize()
pr = cProfile.Profile()
sess.config.target_len = len(sess.committed) + 64
pr.enable(); sess.generate(seed=7); torch.cuda.synchronize(); pr.disable()
st = pstats.Stats(pr); st.sort_stats('tottime').print_stats(25)
