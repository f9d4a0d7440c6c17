import sys; sys.path.insert(0, '/root/repo')
import paper_2511_20975_b200 as P
sp = P.ConfigSpace(2, [(0, 1)], [1.0, 2.0, 3.0], [3.0, 2.0, 1.0])
dev = P.Device(sp)
viable = [sp.index_of(c) for c in ([0, 0], [1, 0], [2, 1])]
q = P.Queue(2, [7], [0.0], [1, 0], [viable])
e = P.Engines([0, 1, 2], [2, 2, 2], [0, 0, 0], [3.0, 2.0, 1.0])
out = P.beam_schedule(dev, q, e, 4)
print(out)
