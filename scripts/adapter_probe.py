"""Per-call latency of the stateless entry points the drop-in adapter uses
(ag_beam_schedule, ag_predict_host) on tiny inputs -- diagnostics."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_20975_b200 as P
from paper_2511_20975_b200._capi import lib, check
sp = P.ConfigSpace.chain(3, 3)
dev = P.Device(sp)
q = P.Queue(3, [1, 2, 3], [0.1, 0.2, 0.3], [[1, 0, 0], [3, 1, 0], [1, 0, 0]],
            [np.arange(27, dtype=np.uint32), np.arange(9, 27, dtype=np.uint32), np.arange(0, 27, 2, dtype=np.uint32)])
eng = P.Engines([0, 1, 2], [2, 2, 2], [1, 1, 2], [4.0, 2.0, 1.0])
for _ in range(20):
    P.beam_schedule(dev, q, eng, 4)
t0 = time.perf_counter()
for _ in range(500):
    P.beam_schedule(dev, q, eng, 4)
print("beam_schedule us/call", (time.perf_counter() - t0) / 500 * 1e6)
pred = P.ConfigPredictor(dev)
b = P.AccuracyBatch.generate(sp, P.GenParams(), 1, 5)
viable = np.zeros(64, np.uint32); nv = np.zeros(1, np.int32)
r = P.OracleRouter(0.002)
t = b.c_struct()
for _ in range(20):
    check(lib().ag_predict_host(pred._h, C.byref(t), C.byref(r), None, C.c_double(1e9), viable.ctypes.data, 64, nv.ctypes.data, None, None, None, None))
t0 = time.perf_counter()
for _ in range(500):
    check(lib().ag_predict_host(pred._h, C.byref(t), C.byref(r), None, C.c_double(1e9), viable.ctypes.data, 64, nv.ctypes.data, None, None, None, None))
print("predict_host us/call", (time.perf_counter() - t0) / 500 * 1e6)
