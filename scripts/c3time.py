"""Config-3 round latency by free-slot class, fast vs general walker (diagnostics).
usage: python scripts/c3time.py [rounds] [beam ...]"""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_20975_b200 as P
from paper_2511_20975_b200 import workloads as W
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 200
beams = [int(b) for b in sys.argv[2:]] or [4, 1]
dev = P.Device(W.config2_space())
for walker in ("auto", "general"):
    os.environ["AG_SCHED_WALKER"] = walker
    for beam in beams:
        c3 = W.Config3(dev, inflight=10000, rounds=rounds + 10, seed=1, beam=beam)
        rows = []
        def cb(rd, a):
            if rd >= 10:
                t = c3.sess.round_timing()
                rows.append((W.config3_engines(rd, 1, [1] * 8)[1], c3.sess.last_round_us(), float(t.sum()), *t))
        lat, h, _ = c3.run(on_round=cb)
        r = np.asarray(rows)
        line = f"{walker:8s} B={beam} hash {h:016x} all p50 {np.percentile(r[:,1],50):7.1f} p99 {np.percentile(r[:,1],99):7.1f} |"
        for f in (1, 8, 64):
            s = r[r[:, 0] == f]
            line += (f" F{f}: capi p50 {np.percentile(s[:,1],50):6.1f} p99 {np.percentile(s[:,1],99):6.1f}"
                     f" dev {np.percentile(s[:,2],50):6.1f}/{np.percentile(s[:,2],99):6.1f}"
                     f" [setup {s[:,3].mean():4.1f} chunk1 {s[:,4].mean():4.1f} walk {s[:,5].mean():5.1f} fin {s[:,6].mean():4.1f}] |")
        print(line, flush=True)
