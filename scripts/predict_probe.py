"""Config-2 chain mode (ConfigPredictor::predict, budget inf) for ncu
captures of k_predict (diagnostics)."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_20975_b200 as P
sp = P.ConfigSpace.chain(5, 8)
dev = P.Device(sp, 0, torch.cuda.current_stream())
t = P.AccuracyBatch.generate(sp, P.GenParams(), 10000, 1).to_device()
pred = P.ConfigPredictor(dev)
for _ in range(3):
    r = pred.predict_batch(t, P.OracleRouter(0.002))
torch.cuda.synchronize()
dev.profile_begin()
for _ in range(5):
    r = pred.predict_batch(t, P.OracleRouter(0.002))
print({k: round(v[0] / v[1] * 1e3, 1) for k, v in dev.profile_end().items()})
