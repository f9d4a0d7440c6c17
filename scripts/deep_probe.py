"""Config 4 on one GPU (8 x 12, 16 requests): enumerate + runtime-cost argmin
over the whole space -- for ncu captures of k_cost_tasks (diagnostics)."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_20975_b200 as P
from paper_2511_20975_b200.scheduler import PER_INPUT_RUNTIME_COST, select_per_input
n, m, R = 8, 12, 16
space = P.ConfigSpace.chain(n, m)
dev = P.Device(space, 0, torch.cuda.current_stream())
truth = P.AccuracyBatch.generate(space, P.GenParams(), R, 1).to_device()
res = dev.route_enumerate(truth, P.OracleRouter())
torch.cuda.synchronize()
mean = [0.05 + float(np.exp(-0.3 + 0.35 * i + 0.5 * 0.25 * 0.25)) for i in range(m)]
load = P.RuntimeCostContext([4] * m, [i % 3 for i in range(m)], [8] * m, mean)
for _ in range(2):
    ch, est = select_per_input(dev, res.indices, res.offsets, PER_INPUT_RUNTIME_COST, load)
torch.cuda.synchronize()
dev.profile_begin()
ch, est = select_per_input(dev, res.indices, res.offsets, PER_INPUT_RUNTIME_COST, load)
print({k: v for k, v in dev.profile_end().items()}, int(res.offsets[-1]))
