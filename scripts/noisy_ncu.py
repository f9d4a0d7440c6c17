import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_20975_b200 as P
sp = P.ConfigSpace.chain(5, 8)
dev = P.Device(sp, 0, torch.cuda.current_stream())
b = P.AccuracyBatch.generate(sp, P.GenParams(), 10000, 1)
t = b.to_device()
r = P.NoisyRouter(0.0, 0.3, 7)
for _ in range(2):
    dev.route_enumerate(t, r, compact=False)
torch.cuda.synchronize()
