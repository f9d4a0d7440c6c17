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


def _sums_dev(res, R):
    """Per-request (count, sum, sum of squares) of a device result, mod 2^64
    (int64 wraps exactly like the reference's uint64 accumulators), plus the
    strict-ascending check inside each request."""
    offs = res.offsets.cpu().numpy().astype(np.int64)
    idx = res.indices
    out = []
    for r in range(R):
        a, b = int(offs[r]), int(offs[r + 1])
        if b == a:
            out.append((0, 0, 0))
            continue
        v = idx[a:b].to(torch.int64) & 0xFFFFFFFF
        if b - a > 1:
            assert bool((v[1:] > v[:-1]).all()), r
        s = int(v.sum().item()) & W.MASK
        q = int((v * v).sum().item()) & W.MASK
        out.append((b - a, s, q))
        del v
    return out


def _digest_of(rows):
    d = 0x5EED
    for c, s, q in rows:
        d = W.mix(d, c, s, q)
    return f"{d:016x}"


def test_config4_full_space_matches_reference_digest():
    """BASELINE config 4 at full size: 8 x 12 chain (429,981,696
    configurations per request), 16 requests, every verdict of the whole
    space (6.9e9) against the unmodified reference's at_index +
    OracleRouter::evaluate loop (accuracy.cpp:227-238, criteria.cpp:93-101):
    the checksum of per-request (count, sum, sum of squares); then the same
    digest from G = 2 / 4 / 8 contiguous canonical-index shards
    (parallel.shard_range, the config-4 sharding), whose member lists must
    lie inside their shard and concatenate in rank order."""
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/ref_bench not built")
    from paper_2511_20975_b200 import parallel as PL

    n, m, R4 = 8, 12, 16
    out = subprocess.run([REF, "route", str(n), str(m), str(R4), "oracle", str(os.cpu_count() or 1),
                          str(SEED)], capture_output=True, text=True, check=True, timeout=1200).stdout
    ref = json.loads(out.strip().splitlines()[-1])
    space = P.ConfigSpace.chain(n, m)
    assert space.size == 429_981_696
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R4, SEED)
    truth = batch.to_device()
    res = dev.route_enumerate(truth, P.OracleRouter())
    torch.cuda.synchronize()
    whole = _sums_dev(res, R4)
    assert sum(c for c, _, _ in whole) == ref["members"]
    assert _digest_of(whole) == ref["digest"]
    del res
    torch.cuda.empty_cache()
    for G in (2, 4, 8):
        acc = [[0, 0, 0] for _ in range(R4)]
        for g in range(G):
            b, e = PL.shard_range(space.size, g, G)
            sres = dev.route_enumerate(truth, P.OracleRouter(), b, e)
            torch.cuda.synchronize()
            offs = sres.offsets.cpu().numpy().astype(np.int64)
            if int(offs[-1]):
                lo = int((sres.indices[: int(offs[-1])].to(torch.int64) & 0xFFFFFFFF).min().item())
                hi = int((sres.indices[: int(offs[-1])].to(torch.int64) & 0xFFFFFFFF).max().item())
                assert b <= lo and hi < e
            for r, (c, s, q) in enumerate(_sums_dev(sres, R4)):
                acc[r][0] += c
                acc[r][1] = (acc[r][1] + s) & W.MASK
                acc[r][2] = (acc[r][2] + q) & W.MASK
            del sres
            torch.cuda.empty_cache()
        assert [tuple(x) for x in acc] == whole, G
        assert _digest_of(acc) == ref["digest"], G


def test_config4_noisy_full_space_matches_reference_digest():
    """Config 4 (8 x 12, 16 requests, 6.9e9 verdicts) with the noisy router of
    config 2 (fp 0, fn 0.3, seed 7): a space above the 2^24 hash-table limit,
    so every verdict takes the per-word hash-chain path of k_route_noise
    (router.cpp:50-57, rng.h:34-51) -- the checksum of per-request
    (count, sum, sum of squares) against the unmodified reference loop."""
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/ref_bench not built")
    n, m, R4 = 8, 12, 16
    out = subprocess.run([REF, "route", str(n), str(m), str(R4), "noisy", str(os.cpu_count() or 1), str(SEED)],
                         capture_output=True, text=True, check=True, timeout=1800).stdout
    ref = json.loads(out.strip().splitlines()[-1])
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    truth = P.AccuracyBatch.generate(space, P.GenParams(), R4, SEED).to_device()
    res = dev.route_enumerate(truth, P.NoisyRouter(0.0, 0.3, 7))
    torch.cuda.synchronize()
    rows = _sums_dev(res, R4)
    assert sum(c for c, _, _ in rows) == ref["members"]
    assert _digest_of(rows) == ref["digest"]
