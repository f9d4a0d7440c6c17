"""Per-round phase breakdown of the config-3 scheduler (diagnostics)."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_20975_b200 as P
from paper_2511_20975_b200 import workloads as W
dev = P.Device(W.config2_space())
c3 = W.Config3(dev, inflight=10000, rounds=int(os.environ.get("C3_ROUNDS", "60")), seed=1, beam=int(sys.argv[1]) if len(sys.argv) > 1 else 4)
rows = []
def cb(rd, a):
    t = c3.sess.round_timing()
    rows.append((rd, W.config3_engines(rd, 1, [1]*8)[1], len(a.triples), a.states_explored, *t,
                 c3.sess.last_round_us(), *(c3.sess.walk_cycles / 1.965e3), *c3.sess.walk_counts, *c3.sess.chunk_us, c3.sess.producers_after_walk_us, *c3.sess.host_timing()))
lat, h, _ = c3.run(on_round=cb)
print("hash %016x" % h)
for r, l in zip(rows, lat):
    print("rd %3d F %2d T %2d expl %7d | setup %6.1f chunk1 %6.1f walk %6.1f fin %6.1f | capi %7.1f | "
          "find %6.1f build %6.1f rank %6.1f adopt %6.1f | steps %4d child %5d | chunk ld %5.1f scan %5.1f rec %5.1f hist %5.1f | prod-walk %7.1f | host prep %5.1f launch %5.1f wait %6.1f read %5.1f | py %7.1f" % (*r, l))
