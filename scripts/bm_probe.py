"""Config-4 (chain 8 x 12, 16 requests) runtime-cost argmin: the member-list
path (ag_select_per_input) vs the bitmap path (ag_select_bitmap), CUDA-event
times and the fraction of words the bitmap path's exact pass evaluates;
also config 3 (chain 5 x 8, 10k requests).  Diagnostics."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_20975_b200 as P


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for (n, m, R, router) in ((8, 12, 16, "oracle"), (8, 12, 16, "noisy"), (5, 8, 10000, "oracle"),
                          (5, 8, 10000, "noisy")):
    sp = P.ConfigSpace.chain(n, m)
    dev = P.Device(sp, 0, torch.cuda.current_stream())
    batch = P.AccuracyBatch.generate(sp, P.GenParams(), R, 1)
    rt = P.OracleRouter() if router == "oracle" else P.NoisyRouter(0.0, 0.3, 7)
    res = dev.route_enumerate(batch.to_device(), rt, bitmap=True)
    torch.cuda.synchronize()
    mean = [0.05 + math.exp(-0.3 + 0.35 * i + 0.5 * 0.25 * 0.25) for i in range(m)]
    load = P.RuntimeCostContext([4] * m, [i % 3 for i in range(m)], [8] * m, mean)
    fm = lambda: P.select_per_input(dev, res.indices, res.offsets, P.PER_INPUT_RUNTIME_COST, load,
                                    check_errors=False)
    fb = lambda: P.select_bitmap(dev, res.bitmap, res.counts, 0, sp.size, P.PER_INPUT_RUNTIME_COST, load,
                                 check_errors=False)
    a, b = fm(), fb()
    same = torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    tm, tb = timed(fm), timed(fb)
    P.select_bitmap_stats(dev, True)
    fb()
    words = P.select_bitmap_stats(dev, False)
    total = R * ((sp.size + 31) // 32)
    dev.profile_begin()
    fb()
    prof = dev.profile_end()
    print(f"chain {n}x{m} R={R} {router}: members {int(res.offsets[-1])}, member path {tm:.3f} ms, "
          f"bitmap path {tb:.3f} ms, same={same}, words evaluated {words}/{total} "
          f"({words / total:.4f}), profile {prof}", flush=True)
    del res, dev
    torch.cuda.empty_cache()
