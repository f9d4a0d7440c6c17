"""Learned-router enumerate (ag_route_linear) on config 2: per-kernel device
times and tensor throughput -- diagnostics."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_20975_b200 as P
sp = P.ConfigSpace.chain(5, 8)
dev = P.Device(sp, 0, torch.cuda.current_stream())
R, D = 10000, 128
g = torch.Generator(device="cuda").manual_seed(1)
emb = torch.randn(R, D, device="cuda", generator=g).to(torch.bfloat16)
heads = (torch.randn(sp.size, D, device="cuda", generator=g) / D ** 0.5).to(torch.bfloat16)
bias = torch.randn(sp.size, device="cuda", generator=g) * 0.1 - 0.2
res = dev.route_linear(emb, heads, bias, compact=False) if False else None
probe = dev.route_linear(emb, heads, bias, capacity=1)
torch.cuda.synchronize()
tot = int(probe.offsets[-1])
out = dev.alloc_route(R, 0, sp.size, tot)
for _ in range(3):
    dev.route_linear(emb, heads, bias, out=out)
torch.cuda.synchronize()
dev.profile_begin()
for _ in range(5):
    dev.route_linear(emb, heads, bias, out=out)
prof = dev.profile_end()
flop = 2.0 * R * sp.size * D
ms = prof["k_linear_score"][0] / prof["k_linear_score"][1]
print("members", tot, {k: round(v[0] / v[1] * 1e3, 1) for k, v in prof.items()},
      "TFLOP/s %.1f" % (flop / (ms / 1e3) / 1e12))
