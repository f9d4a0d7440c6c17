"""Config-3 rounds for an ncu capture of k_sched_round (round 6 is F = 64).
usage: python scripts/sched_ncu.py [rounds] [beam]"""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20975_b200 as P
from paper_2511_20975_b200 import workloads as W
dev = P.Device(W.config2_space())
c3 = W.Config3(dev, inflight=10000, rounds=int(sys.argv[1]) if len(sys.argv) > 1 else 8, seed=1,
               beam=int(sys.argv[2]) if len(sys.argv) > 2 else 4)
lat, h, _ = c3.run()
print("rounds", len(lat), "hash %016x" % h)
