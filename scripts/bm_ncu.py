"""ncu target: one ag_select_bitmap over config 4 (chain 8 x 12, 16
requests) and one over config 3 (chain 5 x 8, 10k requests), oracle router
(diagnostics)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_20975_b200 as P

for (n, m, R) in ((8, 12, 16), (5, 8, 10000)):
    sp = P.ConfigSpace.chain(n, m)
    dev = P.Device(sp, 0, torch.cuda.current_stream())
    batch = P.AccuracyBatch.generate(sp, P.GenParams(), R, 1)
    res = dev.route_enumerate(batch.to_device(), P.OracleRouter(), bitmap=True, compact=False)
    mean = [0.05 + math.exp(-0.3 + 0.35 * i + 0.5 * 0.25 * 0.25) for i in range(m)]
    load = P.RuntimeCostContext([4] * m, [i % 3 for i in range(m)], [8] * m, mean)
    P.select_bitmap(dev, res.bitmap, res.counts, 0, sp.size, P.PER_INPUT_RUNTIME_COST, load)
    torch.cuda.synchronize()
    del res, dev
    torch.cuda.empty_cache()
