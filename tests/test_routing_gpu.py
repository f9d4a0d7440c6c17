"""Routing parity (enumerate mode): the CUDA path through the C ABI against
the reference's golden bitmaps and the C oracle restatement.  Bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _hex_words(h):
    return np.array([int(h[i:i + 8], 16) for i in range(0, len(h), 8)], np.uint32)


def _members(words, count):
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")
    return np.nonzero(bits)[0][:count].astype(np.uint32)


def _oracle_tb(space, batch):
    return O.TruthBatch(space.n, space.m, [batch.seeds_of(r) for r in range(batch.n_requests)],
                        [batch.removed_of(r) for r in range(batch.n_requests)], batch.request_ids)


def _orouter(router):
    return O.Router(router.kind, router.fp, router.fn, router.noise_seed, 0.0)


def _check_against_oracle(dev, space, batch, router, begin=0, end=None, force_top=False):
    end = space.size if end is None else end
    res = dev.route_enumerate(batch.to_device(), router, begin, end, force_top=force_top, bitmap=True)
    torch.cuda.synchronize()
    counts = res.counts.cpu().numpy()
    offs = res.offsets.cpu().numpy()
    idx = res.indices.cpu().numpy().view(np.uint32)
    bm = res.bitmap.cpu().numpy().view(np.uint32)
    tb = _oracle_tb(space, batch)
    for r in range(batch.n_requests):
        cnt, words = O.enumerate_bitmap(tb, _orouter(router), r, begin, end, force_top)
        assert counts[r] == cnt, (r, counts[r], cnt)
        assert np.array_equal(bm[r, : len(words)], words), r
        want = _members(words, cnt) + np.uint32(begin)
        assert np.array_equal(idx[offs[r]:offs[r + 1]], want), r
    assert offs[-1] == counts.sum()


def test_golden_router_bitmaps(golden):
    rows = golden("router.json")
    for r in rows:
        n, m = r["n"], r["m"]
        space = P.ConfigSpace.chain(n, m)
        dev = P.Device(space)
        batch = P.AccuracyBatch.from_lists(n, [r["seeds"]], [r["removed"]], [r["id"]])
        for router, key, cnt_key in ((P.OracleRouter(), "oracle_bitmap", "oracle_count"),
                                     (P.NoisyRouter(r["fp"], r["fn"], r["noise_seed"]),
                                      "noisy_bitmap", "noisy_count")):
            res = dev.route_enumerate(batch.to_device(), router, bitmap=True)
            torch.cuda.synchronize()
            want = _hex_words(r[key])
            got = res.bitmap.cpu().numpy().view(np.uint32)[0, : len(want)]
            assert np.array_equal(got, want), (n, m, r["id"], key)
            assert int(res.counts[0]) == r[cnt_key]
            assert np.array_equal(res.indices[: r[cnt_key]].cpu().numpy().view(np.uint32),
                                  _members(want, r[cnt_key]))


@pytest.mark.parametrize("n,m,R", [(1, 2, 7), (1, 40, 9), (2, 3, 50), (3, 3, 1000), (3, 4, 300),
                                   (4, 3, 200), (5, 8, 600), (6, 5, 40), (7, 3, 90), (9, 2, 64),
                                   (12, 2, 20), (14, 3, 2), (17, 2, 3)])
@pytest.mark.parametrize("noisy", [False, True])
def test_enumerate_matches_oracle(n, m, R, noisy):
    space = P.ConfigSpace.chain(n, m)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=1 + n * m)
    dev = P.Device(space)
    router = P.NoisyRouter(0.07, 0.3, 7 + n) if noisy else P.OracleRouter()
    _check_against_oracle(dev, space, batch, router)


def test_violations_removed_lists():
    space = P.ConfigSpace.chain(4, 4)  # 256 configs, removals allowed
    batch = P.AccuracyBatch.generate(space, P.GenParams(violation_rate=0.08), 80, seed=5)
    assert batch.removed.size > 0
    dev = P.Device(space)
    for router in (P.OracleRouter(), P.NoisyRouter(0.2, 0.1, 3)):
        _check_against_oracle(dev, space, batch, router)


def test_force_top_and_edge_sets():
    space = P.ConfigSpace.chain(3, 5)
    seeds = [[], [[4, 4, 4]], [[0, 0, 0]], [[1, 0, 3], [0, 2, 0], [3, 3, 0]]]
    removed = [[], [], [space.size - 2, 0], []]
    batch = P.AccuracyBatch.from_lists(3, seeds, removed)
    dev = P.Device(space)
    for ft in (False, True):
        for router in (P.OracleRouter(), P.NoisyRouter(0.0, 1.0, 9), P.NoisyRouter(1.0, 0.0, 9)):
            _check_against_oracle(dev, space, batch, router, force_top=ft)


@pytest.mark.parametrize("n,m", [(5, 8), (4, 6), (6, 4)])
def test_seed_counts_on_the_phase_pattern_path(n, m):
    """Hand-built accurate sets with 0..6 seeds (the generator emits <= 2, the
    ABI takes any seed CSR) on spaces where K1 takes its phase-pattern path
    (M*M >= 32): the seed-subset tables (<= 2 seeds), the per-seed tests (3-4)
    and the 2-D fallback (> 4), over full and ragged ranges."""
    space = P.ConfigSpace.chain(n, m)
    rng = np.random.default_rng(n * 100 + m)
    seeds = []
    for k in (0, 1, 2, 2, 3, 4, 5, 6, 1, 2):
        seeds.append([[int(d) for d in rng.integers(0, m, n)] for _ in range(k)])
    batch = P.AccuracyBatch.from_lists(n, seeds, [[] for _ in seeds])
    dev = P.Device(space)
    for a, b in ((0, space.size), (3, space.size - 5), (1024, min(space.size, 70000))):
        _check_against_oracle(dev, space, batch, P.OracleRouter(), a, b)


def test_subranges_concatenate_to_full_range():
    space = P.ConfigSpace.chain(5, 7)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), 40, seed=9)
    dev = P.Device(space)
    router = P.NoisyRouter(0.01, 0.3, 5)
    full = dev.route_enumerate(batch.to_device(), router)
    torch.cuda.synchronize()
    cuts = [0, 1, 33, 1000, 4095, 9999, space.size]
    parts = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        _check_against_oracle(dev, space, batch, router, a, b)
        res = dev.route_enumerate(batch.to_device(), router, a, b)
        torch.cuda.synchronize()
        parts.append((res.counts.cpu().numpy(), res.offsets.cpu().numpy(),
                      res.indices.cpu().numpy().view(np.uint32)))
    fo = full.offsets.cpu().numpy()
    fi = full.indices.cpu().numpy().view(np.uint32)
    for r in range(batch.n_requests):
        cat = np.concatenate([p[2][p[1][r]:p[1][r + 1]] for p in parts])
        assert np.array_equal(cat, fi[fo[r]:fo[r + 1]])


def test_deep_space_range_8x12():
    """BASELINE config 4 shape: 8 agents x 12 tiers, a 3M-index window."""
    space = P.ConfigSpace.chain(8, 12)
    assert space.size == 12 ** 8
    batch = P.AccuracyBatch.generate(space, P.GenParams(), 4, seed=1)
    dev = P.Device(space)
    lo = space.size // 3
    for router in (P.OracleRouter(), P.NoisyRouter(0.05, 0.3, 7)):
        _check_against_oracle(dev, space, batch, router, lo, lo + 3_000_000 + 17)


def test_deep_space_long_window_multi_slice_scan():
    """More than 4096 32-word groups per request: the sliced group scan
    (k_chunk_partial / k_chunk_scan_slices) instead of the warp scan."""
    space = P.ConfigSpace.chain(8, 12)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), 3, seed=5)
    dev = P.Device(space)
    lo = space.size // 5 + 3
    _check_against_oracle(dev, space, batch, P.OracleRouter(), lo, lo + 9_000_000 + 13)


def test_host_path_and_capacity():
    space = P.ConfigSpace.chain(4, 6)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), 100, seed=2)
    dev = P.Device(space)
    router = P.OracleRouter()
    res = dev.route_enumerate_host(batch, router)
    d = dev.route_enumerate(batch.to_device(), router)
    torch.cuda.synchronize()
    assert np.array_equal(res.counts, d.counts.cpu().numpy().astype(np.uint64))
    assert np.array_equal(res.indices, d.indices[: int(d.offsets[-1])].cpu().numpy().view(np.uint32))
    with pytest.raises(P.ValidationError):
        dev.route_enumerate_host(batch, router, capacity=10)
    # device path: overflow flag, nothing written past capacity
    out = dev.alloc_route(batch.n_requests, 0, space.size, 10)
    dev.route_enumerate(batch.to_device(), router, out=out)
    torch.cuda.synchronize()
    assert int(out["overflow"][0]) == 1


def test_empty_inputs():
    space = P.ConfigSpace.chain(3, 3)
    dev = P.Device(space)
    empty = P.AccuracyBatch.from_lists(3, [], [])
    res = dev.route_enumerate_host(empty, P.OracleRouter())
    assert res.offsets[0] == 0 and len(res.indices) == 0
    batch = P.AccuracyBatch.generate(space, P.GenParams(), 5, seed=1)
    res = dev.route_enumerate(batch.to_device(), P.OracleRouter(), 4, 4)
    torch.cuda.synchronize()
    assert res.counts.sum().item() == 0
    with pytest.raises(P.ValidationError):
        dev.route_enumerate(batch.to_device(), P.OracleRouter(), 5, 4)
    with pytest.raises(P.ValidationError):
        dev.route_enumerate(batch.to_device(), P.NoisyRouter(1.5, 0, 1))


def test_reference_enumerate_members_guard():
    space = P.ConfigSpace.chain(2, 3)
    assert P.enumerate_members(space, [[1, 0]]) == [[1, 0], [1, 1], [1, 2], [2, 0], [2, 1], [2, 2]]
    with pytest.raises(P.ValidationError):
        P.enumerate_members(P.ConfigSpace.chain(7, 4), [[0] * 7])


@pytest.mark.parametrize("shift", [1, 2, 3])
@pytest.mark.parametrize("cap_cut", [0, 1, 5, 777])
def test_compaction_unaligned_output_and_partial_capacity(shift, cap_cut):
    """k_route_compact writes 16-byte vectors at the output's own phase: an
    output pointer off 16-byte alignment and a capacity that ends inside a
    vector must still give exactly the canonical members up to capacity and
    leave everything past it untouched."""
    space = P.ConfigSpace.chain(5, 4)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), 37, seed=11)
    dev = P.Device(space)
    router = P.OracleRouter()
    full = dev.route_enumerate(batch.to_device(), router)
    torch.cuda.synchronize()
    total = int(full.offsets[-1])
    want = full.indices[:total].clone()
    cap = total - cap_cut
    sentinel = -7
    big = torch.full((cap + shift + 64,), sentinel, dtype=torch.int32, device=want.device)
    out = dev.alloc_route(batch.n_requests, 0, space.size, cap)
    out["indices"] = big[shift:]
    out["capacity"] = cap
    dev.route_enumerate(batch.to_device(), router, out=out)
    torch.cuda.synchronize()
    got = big[shift:shift + cap]
    assert torch.equal(got, want[:cap])
    assert int((big[:shift] != sentinel).sum()) == 0
    assert int((big[shift + cap:] != sentinel).sum()) == 0
    assert int(out["overflow"][0]) == (1 if cap_cut else 0)
