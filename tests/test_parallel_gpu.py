"""The sharded routing path's device side (config 4 sharding, SURVEY.md
§8(e)) on one GPU: G contiguous canonical-index shards are routed, reduced
to 32-byte records by ag_shard_records, stacked as the all-gather would
deliver them, and merged by ag_merge_records for every rank.  The merge must
equal the whole space: global counts, each rank's global offsets (members
below its shard), and the runtime-cost choice of select_per_input_config
(workload.cpp:149-176) over the whole accurate set, bit-exact (index and
fp64 estimate)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from paper_2511_20975_b200 import parallel as PL  # noqa: E402


@pytest.mark.parametrize("bitmap", [False, True])
@pytest.mark.parametrize("n,m,R,G", [(5, 8, 300, 4), (4, 5, 200, 3), (3, 4, 64, 8), (8, 12, 3, 4)])
def test_shard_records_merge_equals_whole_space(n, m, R, G, bitmap):
    """bitmap: the shard records come straight from each shard's verdict
    bitmap (ag_select_bitmap over [begin, end)) instead of its members."""
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=5 + n)
    truth = batch.to_device()
    mean = [0.05 + math.exp(-0.3 + 0.35 * i + 0.5 * 0.25 * 0.25) for i in range(m)]
    load = P.RuntimeCostContext([4] * m, [i % 3 for i in range(m)], [8] * m, mean)
    whole = dev.route_enumerate(truth, P.OracleRouter())
    w_ch, w_est = P.select_per_input(dev, whole.indices, whole.offsets, P.PER_INPUT_RUNTIME_COST, load)
    w_counts = whole.counts.cpu().numpy().astype(np.int64)
    w_offs = whole.offsets.cpu().numpy()
    w_idx = whole.indices.cpu().numpy().view(np.uint32)
    recs, ranges = [], []
    for g in range(G):
        b, e = PL.shard_range(space.size, g, G)
        res = dev.route_enumerate(truth, P.OracleRouter(), b, e, bitmap=bitmap)
        recs.append(PL.shard_records(dev, res, R, load, b, e))
        ranges.append(b)
        del res
    gathered = torch.stack(recs)
    for rank in range(G):
        total, before, (be, bc, bi) = PL.merge_device(dev, gathered, rank)
        torch.cuda.synchronize()
        assert np.array_equal(total.cpu().numpy(), w_counts)
        want_before = [int(np.sum(w_idx[w_offs[r]:w_offs[r + 1]] < ranges[rank])) for r in range(R)]
        assert before.cpu().numpy().tolist() == want_before
        assert np.array_equal(bi.cpu().numpy().astype(np.uint32), w_ch.cpu().numpy().view(np.uint32))
        assert np.array_equal(be.cpu().numpy(), w_est.cpu().numpy())


def test_sharded_path_world1_matches_whole_space():
    """route_space_sharded with one rank (no collective) is the whole space."""
    space = P.ConfigSpace.chain(5, 8)
    dev = P.Device(space)
    R = 200
    truth = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=9).to_device()
    load = P.RuntimeCostContext([4] * 8, [i % 3 for i in range(8)], [8] * 8, [0.5 + 0.25 * i for i in range(8)])
    for out in (None, dev.alloc_route(R, 0, space.size, R * space.size, bitmap=True)):
        res, total, before, (be, bc, bi) = PL.route_space_sharded(dev, truth, P.OracleRouter(), 0, 1, load,
                                                                  out=out)
        ch, est = P.select_per_input(dev, res.indices, res.offsets, P.PER_INPUT_RUNTIME_COST, load)
        torch.cuda.synchronize()
        assert np.array_equal(total.cpu().numpy(), res.counts.cpu().numpy().astype(np.int64))
        assert (before.cpu().numpy() == 0).all()
        assert np.array_equal(bi.cpu().numpy().astype(np.uint32), ch.cpu().numpy().view(np.uint32))
        assert np.array_equal(be.cpu().numpy(), est.cpu().numpy())


def test_async_select_errors_latch_until_synchronize():
    """ag_select_per_input is asynchronous: the reference's ValidationError
    (a member tier missing from the load context) surfaces at the next
    synchronisation and is then cleared."""
    space = P.ConfigSpace.chain(2, 3)
    dev = P.Device(space)
    mem = torch.tensor([0, 4, 8], dtype=torch.int32, device="cuda")
    offs = torch.tensor([0, 3], dtype=torch.int64, device="cuda")
    bad = P.RuntimeCostContext([0, 0, 0], [0, 0, 0], [1, 1, 0], [1.0, 1.0, 1.0])
    P.select_per_input(dev, mem, offs, P.PER_INPUT_RUNTIME_COST, bad, check_errors=False)
    with pytest.raises(P.ValidationError):
        dev.synchronize()
    dev.synchronize()  # cleared
    good = P.RuntimeCostContext([0, 0, 0], [0, 0, 0], [1, 1, 1], [1.0, 1.0, 1.0])
    ch, _ = P.select_per_input(dev, mem, offs, P.PER_INPUT_RUNTIME_COST, good)
    assert int(ch[0]) == 0
