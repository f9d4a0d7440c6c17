"""Config 4 step breakdown on one GPU (diagnostics): host wall time of each
part of parallel.route_space_sharded."""
import os, sys, time; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_20975_b200 as P
from paper_2511_20975_b200 import parallel as PL
from paper_2511_20975_b200.scheduler import PER_INPUT_RUNTIME_COST, select_per_input
n, m, R = 8, 12, 16
space = P.ConfigSpace.chain(n, m)
dev = P.Device(space, 0, torch.cuda.current_stream())
truth = P.AccuracyBatch.generate(space, P.GenParams(), R, 1).to_device(torch.device("cuda", 0))
router = P.OracleRouter()
probe = dev.route_enumerate(truth, router, 0, space.size, compact=False)
torch.cuda.synchronize()
out = dev.alloc_route(R, 0, space.size, int(probe.offsets[-1]))
mean = [0.05 + float(np.exp(-0.3 + 0.35 * i + 0.5 * 0.25 * 0.25)) for i in range(m)]
load = P.RuntimeCostContext([4] * m, [i % 3 for i in range(m)], [8] * m, mean)
for it in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    res = dev.route_enumerate(truth, router, 0, space.size, out=out)
    t.append(time.perf_counter())
    counts = res.counts.cpu().numpy()
    t.append(time.perf_counter())
    ch, est = select_per_input(dev, res.indices, res.offsets, PER_INPUT_RUNTIME_COST, load)
    t.append(time.perf_counter())
    bi = ch.cpu().numpy(); be = est.cpu().numpy()
    t.append(time.perf_counter())
    r2 = PL.route_space_sharded(dev, truth, router, 0, 1, load, out=out)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("enum-launch %.3f  counts(sync) %.3f  select %.3f  ch/est cpu %.3f | whole sharded step %.3f ms" % tuple(d))
