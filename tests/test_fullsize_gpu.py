"""BASELINE config 2 at full size (5 x 8, 10,000 requests, seed 1) against
the unmodified reference (oracle/_ref/ref_bench route: the at_index +
RouterBackend::evaluate loop, criteria.cpp:93-101): every request's member
list is strictly ascending and inside the space, and the checksum of
per-request checksums -- D = mix({D, count, sum of indices, sum of squares})
in request order -- equals the reference's, for the oracle router and the
noisy router of config 2 (fp 0, fn 0.3, seed 7)."""
import json
import os
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from paper_2511_20975_b200 import workloads as W  # noqa: E402

REF = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "ref_bench")
R, SEED = 10_000, 1


def digest(counts, offsets, idx):
    u = idx.astype(np.uint64)
    starts = offsets[:-1].astype(np.int64)
    nz = counts > 0
    sums = np.zeros(len(counts), np.uint64)
    sqs = np.zeros(len(counts), np.uint64)
    if nz.any():
        sums[nz] = np.add.reduceat(u, starts[nz])
        sqs[nz] = np.add.reduceat(u * u, starts[nz])
    d = 0x5EED
    for r in range(len(counts)):
        d = W.mix(d, int(counts[r]), int(sums[r]), int(sqs[r]))
    return f"{d:016x}"


@pytest.mark.parametrize("router", ["oracle", "noisy"])
def test_config2_full_batch_matches_reference_digest(router):
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/ref_bench not built")
    out = subprocess.run([REF, "route", "5", "8", str(R), router, str(os.cpu_count() or 1), str(SEED)],
                         capture_output=True, text=True, check=True, timeout=600).stdout
    ref = json.loads(out.strip().splitlines()[-1])
    space = W.config2_space()
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, SEED)
    rt = P.OracleRouter() if router == "oracle" else P.NoisyRouter(0.0, 0.3, 7)
    res = dev.route_enumerate(batch.to_device(), rt)
    torch.cuda.synchronize()
    counts = res.counts.cpu().numpy()
    offsets = res.offsets.cpu().numpy()
    idx = res.indices.cpu().numpy().view(np.uint32)[: int(offsets[-1])]
    assert int(offsets[-1]) == ref["members"]
    assert (np.diff(offsets.astype(np.int64)) == counts.astype(np.int64)).all()
    # strictly ascending inside each request, every index inside the space
    assert int(idx.max()) < space.size
    d = np.diff(idx.astype(np.int64))
    bounds = offsets[1:-1].astype(np.int64) - 1  # last position of each request but the final
    ok = d > 0
    ok[bounds[(bounds >= 0) & (bounds < len(d))]] = True
    assert ok.all()
    assert digest(counts, offsets, idx) == ref["digest"]
