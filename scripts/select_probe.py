"""Config-3 re-cost + argmin (ag_select_per_input) over the exhaustive
accurate sets of the 10k config-2 requests, and chain-mode predict over the
same batch: target for ncu captures of k_cost_* and k_predict (diagnostics)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_20975_b200 as P

sp = P.ConfigSpace.chain(5, 8)
dev = P.Device(sp, 0, torch.cuda.current_stream())
batch = P.AccuracyBatch.generate(sp, P.GenParams(), 10000, 1)
truth = batch.to_device()
res = dev.route_enumerate(truth, P.OracleRouter())
mean = [0.05 + math.exp((-0.3 + 0.35 * i) + 0.5 * 0.25 * 0.25) for i in range(8)]
load = P.RuntimeCostContext([4] * 8, [i % 3 for i in range(8)], [8] * 8, mean)
for _ in range(3):
    P.select_per_input(dev, res.indices, res.offsets, P.PER_INPUT_RUNTIME_COST, load, check_errors=False)
pred = P.ConfigPredictor(dev)
for _ in range(3):
    pred.predict_batch(truth, P.OracleRouter(0.002))
dev.profile_begin()
P.select_per_input(dev, res.indices, res.offsets, P.PER_INPUT_RUNTIME_COST, load, check_errors=False)
pred.predict_batch(truth, P.OracleRouter(0.002))
prof = dev.profile_end()
print({k: (round(v[0] * 1e3, 1), v[1]) for k, v in prof.items()})
