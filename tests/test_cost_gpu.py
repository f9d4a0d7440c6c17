"""Runtime-cost re-cost + argmin (select_per_input_config, estimate_completion)
and snapshot_load's queued_ahead on the GPU, against the reference's golden
selections (tests/golden/workload.json) and the C oracle.  Bit-exact: chosen
configuration and its fp64 estimate."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _csr(lists, dev):
    offs = np.zeros(len(lists) + 1, np.int64)
    for i, v in enumerate(lists):
        offs[i + 1] = offs[i] + len(v)
    mem = np.concatenate([np.asarray(v, np.uint32) for v in lists]) if offs[-1] else np.zeros(1, np.uint32)
    return (torch.from_numpy(mem.view(np.int32)).to(dev), torch.from_numpy(offs).to(dev))


def test_golden_selections(golden):
    rows = golden("workload.json")
    groups = {}
    for w in rows:
        groups.setdefault((w["n"], w["m"]), []).append(w)
    for (n, m), ws in groups.items():
        space = P.ConfigSpace(n, [(i - 1, i) for i in range(1, n)], ws[0]["cost"],
                              [8.0 / 1.5 ** i for i in range(m)])
        dev = P.Device(space)
        mem, offs = _csr([w["members"] for w in ws], dev.torch_device)
        ch, _ = P.select_per_input(dev, mem, offs, P.PER_INPUT_STATIC)
        assert ch.cpu().numpy().view(np.uint32).tolist() == [w["static_pick"] for w in ws]
        for i, w in enumerate(ws):  # one load context per request
            ctx = P.RuntimeCostContext(w["occupancy"], w["queued_ahead"], w["slots"], w["mean"])
            ch, est = P.select_per_input(dev, mem[int(offs[i]):int(offs[i + 1])],
                                         offs[i:i + 2] - offs[i], P.PER_INPUT_RUNTIME_COST, ctx)
            assert int(ch[0]) == w["runtime_pick"]
            assert float(est[0]) == w["runtime_est"]


@pytest.mark.parametrize("n,m,R", [(5, 8, 300), (3, 4, 500), (4, 3, 400)])
def test_matches_oracle_with_ties(n, m, R):
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=3)
    res = dev.route_enumerate(batch.to_device(), P.OracleRouter())
    torch.cuda.synchronize()
    offs = res.offsets.cpu().numpy()
    idx = res.indices.cpu().numpy().view(np.uint32)
    rng = np.random.default_rng(m)
    for trial in range(3):
        slots = rng.integers(1, 9, m).tolist()
        occ = [int(rng.integers(0, s + 1)) for s in slots]
        queued = rng.integers(0, 3 if trial == 0 else 50, m).tolist()
        mean = [0.05 + math.exp(-0.3 + 0.4 * i + 0.5 * 0.25 * 0.25) for i in range(m)]
        ctx = P.RuntimeCostContext(occ, queued, slots, mean)
        ch, est = P.select_per_input(dev, res.indices, res.offsets, P.PER_INPUT_RUNTIME_COST, ctx)
        ch = ch.cpu().numpy().view(np.uint32)
        est = est.cpu().numpy()
        for r in range(0, R, 7):
            members = idx[offs[r]:offs[r + 1]]
            want, west = O.select_per_input(n, m, space.cost, occ, queued, slots, mean, 1, members)
            assert ch[r] == want and est[r] == west


def test_validation():
    space = P.ConfigSpace.chain(2, 3)
    dev = P.Device(space)
    mem, offs = _csr([[0, 4, 8]], dev.torch_device)
    with pytest.raises(P.ValidationError):  # tier 2 has no slots
        P.select_per_input(dev, mem, offs, P.PER_INPUT_RUNTIME_COST,
                           P.RuntimeCostContext([0, 0, 0], [0, 0, 0], [1, 1, 0], [1.0, 1.0, 1.0]))
    with pytest.raises(P.ValidationError):  # no context
        P.select_per_input(dev, mem, offs, P.PER_INPUT_RUNTIME_COST, None)
    mem, offs = _csr([[]], dev.torch_device)
    with pytest.raises(P.ValidationError):  # empty set
        P.select_per_input(dev, mem, offs, P.PER_INPUT_STATIC)


def test_queued_ahead_matches_definition():
    from paper_2511_20975_b200 import workloads as W
    dev = P.Device(W.config2_space())
    c3 = W.Config3(dev, inflight=500, rounds=5, seed=2, beam=4)
    qa = c3.sess.queued_ahead()
    want = [0] * 8
    n = 5
    for s, st in c3.stages.items():
        for a in range(n):
            if st[a] == 1:
                v = c3.sess.viable(s)
                for mdl in set(((v // 8 ** (n - 1 - a)) % 8).tolist()):
                    want[mdl] += 1
    assert qa == want


@pytest.mark.parametrize("n,m", [(8, 12), (25, 2), (26, 2), (32, 2), (4, 200)])
def test_prefix_table_suffix_lengths(n, m):
    """The prefix-table split (k digits tabulated, N - k folded per member)
    for every suffix length the kernel specialises and the generic one:
    random sorted member lists over the whole space against the oracle."""
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    rng = np.random.default_rng(n * 1000 + m)
    S = m ** n
    lists = [np.unique(rng.integers(0, S, int(rng.integers(1, 3000)), dtype=np.uint64)).astype(np.uint32)
             for _ in range(24)]
    lists.append(np.arange(min(S, 5000), dtype=np.uint32))  # a dense run (many ties)
    mem, offs = _csr(lists, dev.torch_device)
    slots = rng.integers(1, 9, m).tolist()
    occ = [int(rng.integers(0, s + 1)) for s in slots]
    queued = rng.integers(0, 5, m).tolist()
    mean = [0.05 + math.exp(-0.3 + 0.01 * i) for i in range(m)]
    ctx = P.RuntimeCostContext(occ, queued, slots, mean)
    for kind in (P.PER_INPUT_STATIC, P.PER_INPUT_RUNTIME_COST):
        ch, est = P.select_per_input(dev, mem, offs, kind, ctx if kind == P.PER_INPUT_RUNTIME_COST else None)
        ch = ch.cpu().numpy().view(np.uint32)
        est = est.cpu().numpy()
        for r, members in enumerate(lists):
            want, west = O.select_per_input(n, m, space.cost, occ, queued, slots, mean,
                                            1 if kind == P.PER_INPUT_RUNTIME_COST else 0, members)
            assert ch[r] == want
            if kind == P.PER_INPUT_RUNTIME_COST:
                assert est[r] == west
