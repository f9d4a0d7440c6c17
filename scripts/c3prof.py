import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_20975_b200 as P
from paper_2511_20975_b200 import workloads as W
dev = P.Device(W.config2_space())
c3 = W.Config3(dev, inflight=10000, rounds=40, seed=1, beam=4)
lat, h, a = c3.run()
print(np.percentile(lat, 50))
