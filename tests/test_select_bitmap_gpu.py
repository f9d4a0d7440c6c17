"""select_per_input_config straight from the verdict bitmap (ag_select_bitmap)
against the member-list path (ag_select_per_input, itself pinned to the
reference goldens and the C oracle in test_cost_gpu.py) and the oracle:
bit-exact chosen index and fp64 estimate, static and runtime-cost kinds,
shard ranges that start and end mid-word and mid-prefix, the noisy router,
random loads that reorder the tiers, and the reference's ValidationErrors
(workload.cpp:140-156)."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _route(dev, batch, router, begin=0, end=None):
    return dev.route_enumerate(batch.to_device(), router, begin, end, bitmap=True)


def _loads(m, seed, n=3):
    rng = np.random.default_rng(seed)
    out = []
    for trial in range(n):
        slots = rng.integers(1, 9, m).tolist()
        occ = [int(rng.integers(0, s + 1)) for s in slots]
        queued = rng.integers(0, 3 if trial == 0 else 60, m).tolist()
        if trial == 2:  # unordered means: the cheapest tier is not the lowest
            mean = rng.uniform(0.05, 20.0, m).tolist()
        else:
            mean = [0.05 + math.exp(-0.3 + 0.35 * i + 0.5 * 0.25 * 0.25) for i in range(m)]
        out.append(P.RuntimeCostContext(occ, queued, slots, mean))
    return out


def _both(dev, res, R, begin, end, kind, ctx):
    a = P.select_per_input(dev, res.indices, res.offsets, kind, ctx)
    b = P.select_bitmap(dev, res.bitmap, res.counts[:R], begin, end, kind, ctx)
    return ([t.cpu().numpy() for t in a], [t.cpu().numpy() for t in b])


@pytest.mark.parametrize("n,m,R", [(5, 8, 600), (3, 4, 300), (6, 12, 24), (4, 3, 200), (2, 8, 100),
                                   (16, 2, 40), (3, 40, 30), (9, 5, 6)])
def test_matches_member_path(n, m, R):
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=11)
    res = _route(dev, batch, P.OracleRouter())
    for ctx in _loads(m, n * 100 + m):
        (ca, ea), (cb, eb) = _both(dev, res, R, 0, space.size, P.PER_INPUT_RUNTIME_COST, ctx)
        assert np.array_equal(ca, cb)
        assert np.array_equal(ea.view(np.int64), eb.view(np.int64))
    (ca, _), (cb, _) = _both(dev, res, R, 0, space.size, P.PER_INPUT_STATIC, None)
    assert np.array_equal(ca, cb)


@pytest.mark.parametrize("n,m", [(5, 8), (6, 12)])
def test_noisy_router(n, m):
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    R = 64
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=5)
    res = _route(dev, batch, P.NoisyRouter(0.1, 0.05, 99))
    for ctx in _loads(m, 7):
        (ca, ea), (cb, eb) = _both(dev, res, R, 0, space.size, P.PER_INPUT_RUNTIME_COST, ctx)
        assert np.array_equal(ca, cb)
        assert np.array_equal(ea.view(np.int64), eb.view(np.int64))


@pytest.mark.parametrize("begin_frac,end_frac", [(0.0, 0.5), (0.31, 0.77), (0.5, 1.0)])
def test_shard_ranges_and_records(begin_frac, end_frac):
    n, m, R = 6, 12, 16
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    begin = int(space.size * begin_frac) + (13 if begin_frac else 0)  # mid-word, mid-prefix
    end = int(space.size * end_frac) - (5 if end_frac < 1 else 0)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=21)
    res = _route(dev, batch, P.OracleRouter(), begin, end)
    from paper_2511_20975_b200 import parallel as PL

    for ctx in _loads(m, 3, 2):
        rec_bm = torch.zeros((R, 4), dtype=torch.int64, device=dev.torch_device)
        P.select_bitmap(dev, res.bitmap, res.counts[:R], begin, end, P.PER_INPUT_RUNTIME_COST, ctx,
                        records=rec_bm)
        rec_mem = PL.shard_records(dev, P.RouteResult(res.counts, res.offsets, res.indices, None), R, ctx)
        torch.cuda.synchronize()
        assert torch.equal(rec_bm, rec_mem)
        # non-empty shards also through chosen / est
        counts = res.counts.cpu().numpy()
        if (counts > 0).all():
            (ca, ea), (cb, eb) = _both(dev, res, R, begin, end, P.PER_INPUT_RUNTIME_COST, ctx)
            assert np.array_equal(ca, cb)
            assert np.array_equal(ea.view(np.int64), eb.view(np.int64))


def test_against_oracle():
    n, m, R = 5, 8, 200
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=4)
    res = _route(dev, batch, P.OracleRouter())
    offs = res.offsets.cpu().numpy()
    idx = res.indices.cpu().numpy().view(np.uint32)
    ctx = _loads(m, 9)[1]
    ch, est = P.select_bitmap(dev, res.bitmap, res.counts[:R], 0, space.size, P.PER_INPUT_RUNTIME_COST, ctx)
    ch = ch.cpu().numpy().view(np.uint32)
    est = est.cpu().numpy()
    for r in range(0, R, 9):
        want, west = O.select_per_input(n, m, space.cost, ctx.occupancy, ctx.queued_ahead, ctx.slots, ctx.mean,
                                        1, idx[offs[r]:offs[r + 1]])
        assert ch[r] == want and est[r] == west


def test_pruning_evaluates_few_words():
    """The exact pass touches a small fraction of the words on the config-4
    shape (the bound is what makes the bitmap path cheaper than a member
    read); the result still equals the member path."""
    n, m, R = 7, 12, 4
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=8)
    res = _route(dev, batch, P.OracleRouter())
    ctx = _loads(m, 1, 1)[0]
    P.select_bitmap_stats(dev, True)
    cb, eb = P.select_bitmap(dev, res.bitmap, res.counts[:R], 0, space.size, P.PER_INPUT_RUNTIME_COST, ctx)
    words = P.select_bitmap_stats(dev, False)
    total = R * ((space.size + 31) // 32)
    assert 0 < words < total // 20
    ca, ea = P.select_per_input(dev, res.indices, res.offsets, P.PER_INPUT_RUNTIME_COST, ctx)
    assert torch.equal(ca, cb) and torch.equal(ea, eb)


def test_validation():
    space = P.ConfigSpace.chain(3, 3)
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), 4, seed=2)
    res = _route(dev, batch, P.OracleRouter())
    counts = res.counts[:4]
    with pytest.raises(P.ValidationError):  # a tier without slots, used by some member
        P.select_bitmap(dev, res.bitmap, counts, 0, space.size, P.PER_INPUT_RUNTIME_COST,
                        P.RuntimeCostContext([0, 0, 0], [0, 0, 0], [1, 1, 0], [1.0, 1.0, 1.0]))
    with pytest.raises(P.ValidationError):  # no context
        P.select_bitmap(dev, res.bitmap, counts, 0, space.size, P.PER_INPUT_RUNTIME_COST, None)
    with pytest.raises(P.ValidationError):  # range outside the space
        P.select_bitmap(dev, res.bitmap, counts, 0, space.size + 1, P.PER_INPUT_STATIC, None)
    empty = torch.zeros_like(res.bitmap)
    with pytest.raises(P.ValidationError):  # an empty accurate set
        P.select_bitmap(dev, empty, torch.zeros_like(counts), 0, space.size, P.PER_INPUT_STATIC, None)


@pytest.mark.parametrize("n,m,R", [(5, 8, 300), (6, 12, 8), (3, 4, 100)])
def test_host_entry_point_against_oracle(n, m, R):
    """ag_select_per_input_host (the drop-in adapter's call for
    select_per_input_config): host sets in, choices out, oracle-equal."""
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=13)
    res = _route(dev, batch, P.OracleRouter())
    offs = res.offsets.cpu().numpy()
    idx = res.indices.cpu().numpy().view(np.uint32)
    for kind, ctx in ((P.PER_INPUT_RUNTIME_COST, _loads(m, 17)[2]), (P.PER_INPUT_STATIC, None)):
        ch, est = P.select_per_input_host(dev, batch, kind, ctx)
        for r in range(0, R, max(1, R // 25)):
            if kind == P.PER_INPUT_STATIC:
                want, west = O.select_per_input(n, m, space.cost, [0] * m, [0] * m, [1] * m, [1.0] * m, 0,
                                                idx[offs[r]:offs[r + 1]])
                assert ch[r] == want
            else:
                want, west = O.select_per_input(n, m, space.cost, ctx.occupancy, ctx.queued_ahead, ctx.slots,
                                                ctx.mean, 1, idx[offs[r]:offs[r + 1]])
                assert ch[r] == want and est[r] == west


REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "ref_bench")


@pytest.mark.parametrize("n,m,R", [(5, 8, 2000), (7, 12, 4), (8, 12, 4)])
def test_digest_matches_unmodified_reference(n, m, R):
    """The unmodified reference's select_per_input_config over the exhaustive
    accurate sets (oracle/_ref/ref_bench select: at_index + accurate, the
    (static_cost, models) sort, strict-< scan of estimate_completion) against
    the bitmap path on the same generator output: digest of (chosen index,
    estimate bits) per request.  (8, 12) is the config-4 space at full size
    (4.3e8 configurations per request; 4 of its 16 requests, so that the
    reference's Configuration vectors fit in host memory) and (7, 12) the
    same shape one agent shorter: the prefix bounds prune all but a few
    words there."""
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/ref_bench not built")
    from paper_2511_20975_b200 import workloads as W

    seed = 1
    out = subprocess.run([REF, "select", str(n), str(m), str(R), str(os.cpu_count() or 1), str(seed), "exhaustive"],
                         capture_output=True, text=True, check=True, timeout=900).stdout
    ref = json.loads(out.strip().splitlines()[-1])
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed)
    res = _route(dev, batch, P.OracleRouter())
    mean = [0.05 + math.exp((-0.3 + 0.35 * i) + 0.5 * 0.25 * 0.25) for i in range(m)]
    ctx = P.RuntimeCostContext([4] * m, [i % 3 for i in range(m)], [8] * m, mean)
    ch, est = P.select_bitmap(dev, res.bitmap, res.counts[:R], 0, space.size, P.PER_INPUT_RUNTIME_COST, ctx)
    ch = ch.cpu().numpy().view(np.uint32)
    bits = est.cpu().numpy().view(np.uint64)
    d = 0x5EED
    for r in range(R):
        d = W.mix(d, int(ch[r]), int(bits[r]))
    assert int(res.counts.sum().item()) == ref["configs_costed"]
    assert f"{d:016x}" == ref["digest"]


def test_randomised_spaces_ranges_and_loads():
    """Randomised cross-check of the bitmap path against the member path:
    chain spaces of 2-8 agents and 2-16 tiers, oracle or noisy verdicts,
    random shard ranges (records) and whole-space selections, random loads
    (including negative and tied estimate terms), both policy kinds."""
    rng = np.random.default_rng(2024)
    for case in range(24):
        n = int(rng.integers(2, 9))
        m = int(rng.integers(2, 17))
        while m ** n > 2_000_000:
            n -= 1
        space = P.ConfigSpace.chain(n, m)
        dev = P.Device(space)
        R = int(rng.integers(1, 40))
        batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=int(rng.integers(1, 1 << 30)))
        router = P.OracleRouter() if case % 2 == 0 else P.NoisyRouter(float(rng.uniform(0, 0.2)),
                                                                        float(rng.uniform(0, 0.4)),
                                                                        int(rng.integers(1, 1000)))
        if case % 3 == 2:
            b = int(rng.integers(0, space.size // 2))
            e = int(rng.integers(b + 1, space.size + 1))
        else:
            b, e = 0, space.size
        res = _route(dev, batch, router, b, e)
        slots = rng.integers(1, 9, m).tolist()
        occ = [int(rng.integers(0, s + 1)) for s in slots]
        queued = rng.integers(0, 20, m).tolist()
        mean = (rng.choice([0.5, 1.0, 2.0], m) if case % 4 == 1 else rng.uniform(-1.0, 10.0, m)).tolist()
        ctx = P.RuntimeCostContext(occ, queued, slots, mean)
        for kind, c in ((P.PER_INPUT_RUNTIME_COST, ctx), (P.PER_INPUT_STATIC, None)):
            rec_bm = torch.zeros((R, 4), dtype=torch.int64, device=dev.torch_device)
            P.select_bitmap(dev, res.bitmap, res.counts[:R], b, e, kind, c, check_errors=False, records=rec_bm)
            if kind == P.PER_INPUT_RUNTIME_COST:
                from paper_2511_20975_b200 import parallel as PL

                rec_mem = PL.shard_records(dev, P.RouteResult(res.counts, res.offsets, res.indices, None), R, c)
                torch.cuda.synchronize()
                assert torch.equal(rec_bm, rec_mem), case
            if bool((res.counts[:R] > 0).all()):
                (ca, ea), (cb, eb) = _both(dev, res, R, b, e, kind, c)
                assert np.array_equal(ca, cb), case
                assert np.array_equal(ea.view(np.int64), eb.view(np.int64)), case
