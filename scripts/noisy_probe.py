"""Config 2 with the noisy router (fp 0, fn 0.3, seed 7): per-kernel device
times (live profile) -- diagnostics."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_20975_b200 as P
sp = P.ConfigSpace.chain(5, 8)
dev = P.Device(sp, 0, torch.cuda.current_stream())
b = P.AccuracyBatch.generate(sp, P.GenParams(), 10000, 1)
t = b.to_device()
for name, r in (("oracle", P.OracleRouter()), ("noisy", P.NoisyRouter(0.0, 0.3, 7)),
                ("noisy_fp", P.NoisyRouter(0.05, 0.3, 7))):
    probe = dev.route_enumerate(t, r, compact=False)
    torch.cuda.synchronize()
    out = dev.alloc_route(10000, 0, sp.size, int(probe.offsets[-1]))
    for _ in range(3):
        dev.route_enumerate(t, r, out=out)
    torch.cuda.synchronize()
    dev.profile_begin()
    for _ in range(5):
        dev.route_enumerate(t, r, out=out)
    prof = dev.profile_end()
    print(name, int(out["offsets"][-1]), {k: round(v[0] / v[1] * 1e3, 1) for k, v in prof.items()})
