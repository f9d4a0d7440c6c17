"""Per-stage scheduler parity: beam_schedule on the GPU against the
reference's golden rounds (generate_snapshot corpora, synthetic rounds), the
reference unit-test cases (scheduler_test.cpp), and the C oracle over
multi-round resident sessions with dispatch/complete.  Bit-exact: triples,
occupancy, fp64 utilization/flexibility, skips, states_explored."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

READY = 1
DIAMOND = [(0, 1), (0, 2), (1, 3), (2, 3)]


def _edges_for(n, depth):
    # snapshot / round graphs are chains or the diamond a->{b,c}->d
    if n == 4 and list(depth) == [2, 1, 1, 0]:
        return DIAMOND
    return [(i - 1, i) for i in range(1, n)]


def _run_json_case(dev_cache, j):
    n, m = j["n"], j["m"]
    key = (n, m, tuple(j["graph"]["depth"]))
    if key not in dev_cache:
        sp = P.ConfigSpace(n, _edges_for(n, j["graph"]["depth"]), [1.0 + i for i in range(m)],
                           [8.0 / 1.5 ** i for i in range(m)])
        assert sp.depth.tolist() == j["graph"]["depth"]
        dev_cache[key] = P.Device(sp)
    dev = dev_cache[key]
    reqs, engs = j["requests"], j["engines"]
    q = P.Queue(n, [r["id"] for r in reqs], [r["arrival"] for r in reqs],
                [s for r in reqs for s in r["stages"]], [r["viable"] for r in reqs])
    e = P.Engines([x["model"] for x in engs], [x["slots"] for x in engs],
                  [x["occupancy"] for x in engs], [x["weight"] for x in engs])
    for w, want in j["beam"].items():
        got = P.beam_schedule(dev, q, e, int(w))
        assert [list(t) for t in got.triples] == want["triples"], w
        assert got.occupancy == want["occupancy"]
        assert got.utilization == want["utilization"]
        assert got.flexibility == want["flexibility"]
        assert got.skips == want["skips"]
        assert got.states_explored == want["states_explored"]


def test_golden_snapshots(golden):
    cache = {}
    for seed, rows in golden("snapshots.json").items():
        for j in rows:
            _run_json_case(cache, j)


def test_golden_rounds(golden):
    cache = {}
    for j in golden("rounds.json"):
        _run_json_case(cache, j)


def _eng(models, slots, weights, occ=None):
    return P.Engines(models, slots, occ or [0] * len(models), weights)


def test_reference_unit_cases():
    sp = P.ConfigSpace(1, [], [1.0, 2.0], [2.0, 1.0])
    dev = P.Device(sp)
    # scheduler_test.cpp:108-119 forced skip
    q = P.Queue(1, [1], [0.0], [READY], [[0]])
    out = P.beam_schedule(dev, q, _eng([0, 1], [1, 4], [2.0, 1.0], [1, 0]), 4)
    assert out.triples == [] and out.skips == 1
    # scheduler_test.cpp:143-156 flexibility tie-break 2/3, B=1
    sp2 = P.ConfigSpace(2, [(0, 1)], [1.0, 2.0], [2.0, 1.0])
    dev2 = P.Device(sp2)
    q = P.Queue(2, [1], [0.0], [1, 0], [[0, 1, 3]])
    out = P.beam_schedule(dev2, q, _eng([0, 1], [1, 1], [1.0, 1.0]), 1)
    assert len(out.triples) == 1 and out.triples[0][3] == 0
    assert out.flexibility == pytest.approx(2.0 / 3.0)
    # scheduler_test.cpp:307-315 empty queue
    out = P.beam_schedule(dev2, P.Queue(2, [], [], [], []), _eng([0, 1], [2, 2], [2.0, 1.0]), 4)
    assert out.triples == [] and out.skips == 0 and out.utilization == 0.0
    # scheduler_test.cpp:317-323 duplicate pools
    with pytest.raises(P.ValidationError):
        P.beam_schedule(dev, P.Queue(1, [1], [0.0], [1], [[0]]), _eng([0, 0], [2, 2], [2.0, 1.0]), 4)
    # viable tier without a pool; over capacity; beam width < 1
    with pytest.raises(P.ValidationError):
        P.beam_schedule(dev, P.Queue(1, [1], [0.0], [1], [[1]]), _eng([0], [2], [2.0]), 4)
    with pytest.raises(P.ValidationError):
        P.beam_schedule(dev, P.Queue(1, [1], [0.0], [1], [[0]]),
                        _eng([0, 1], [2, 2], [2.0, 1.0], [3, 0]), 4)
    with pytest.raises(P.ValidationError):
        P.beam_schedule(dev, P.Queue(1, [1], [0.0], [1], [[0]]), _eng([0, 1], [2, 2], [2.0, 1.0]), 0)


def test_reference_diamond_cases():
    # scheduler_test.cpp:121-141: b, c ready after a ran model 0; equal-score
    # alternatives resolve to the smaller triples (mb == 0)
    sp = P.ConfigSpace(4, DIAMOND, [1.0, 2.0], [2.0, 1.0])
    dev = P.Device(sp)
    viable = [sp.index_of(c) for c in ([0, 0, 1, 1], [0, 1, 0, 1])]
    q = P.Queue(4, [1], [0.0], [3, 1, 1, 0], [viable])
    out = P.beam_schedule(dev, q, _eng([0, 1], [4, 4], [2.0, 1.0]), 4)
    assert len(out.triples) == 2 and out.utilization == pytest.approx(3.0)
    assert out.triples[0][3] == 0 and out.triples[1][3] == 1
    # scheduler_test.cpp:158-184: greedy 3.9 vs beam 4.7
    sp3 = P.ConfigSpace(4, DIAMOND, [1.0, 2.1, 4.4], [3.0, 1.7, 0.9])
    dev3 = P.Device(sp3)
    viable = [sp3.index_of([0, b, c, d]) for b in range(3) for c in range(3) for d in range(3)
              if c >= 2 or b >= 1]
    q = P.Queue(4, [1], [0.0], [3, 1, 1, 0], [viable])
    e = _eng([0, 1, 2], [1, 1, 1], [3.0, 1.7, 0.9])
    assert P.beam_schedule(dev3, q, e, 1).utilization == pytest.approx(3.9)
    assert P.beam_schedule(dev3, q, e, 4).utilization == pytest.approx(4.7)


def _oracle_round(n, m, depth, decl, reqs, engines, width):
    qd = O.QueueData(n, m, depth, decl, [r["id"] for r in reqs], [r["arrival"] for r in reqs],
                     [s for r in reqs for s in r["stages"]], [r["viable"] for r in reqs],
                     engines.model, engines.slots, engines.occupancy, engines.weight)
    return O.beam_schedule(qd, width)


@pytest.mark.parametrize("shape,nreq,width,seed", [
    ("chain5x8", 3000, 4, 1), ("chain5x8", 3000, 1, 2), ("diamond4x3", 400, 4, 3),
    ("diamond4x4", 300, 8, 4), ("chain3x3", 500, 2, 5)])
def test_session_multi_round_matches_oracle(shape, nreq, width, seed):
    rng = np.random.default_rng(seed)
    if shape.startswith("chain"):
        n, m = (int(x) for x in shape[5:].split("x"))
        edges = [(i - 1, i) for i in range(1, n)]
    else:
        n, m = 4, int(shape.split("x")[1])
        edges = DIAMOND
    sp = P.ConfigSpace(n, edges, [1.5 ** i for i in range(m)], [8.0 / 1.5 ** i for i in range(m)])
    dev = P.Device(sp)
    batch = P.AccuracyBatch.generate(sp, P.GenParams(), nreq, seed)
    if sp.size <= 4096:  # exhaustive viable sets
        res = dev.route_enumerate_host(batch, P.OracleRouter())
        viable = [res.indices[res.offsets[r]:res.offsets[r + 1]].copy() for r in range(nreq)]
    else:  # chain-mode predictor sets
        pred = P.ConfigPredictor(dev)
        pr = pred.predict_batch(batch.to_device(), P.OracleRouter(0.001))
        torch.cuda.synchronize()
        nv = pr.n_viable.cpu().numpy()
        vv = pr.viable.cpu().numpy().view(np.uint32)
        viable = [vv[r, : nv[r]].copy() for r in range(nreq)]
    depth, decl = sp.depth.tolist(), sp.decl.tolist()
    pred_mask = [sum(1 << a for a, b in edges if b == x) for x in range(n)]
    reqs = []
    for r in range(nreq):
        stages = [1 if pred_mask[a] == 0 else 0 for a in range(n)]
        reqs.append(dict(id=int(10_000 + r), arrival=float(r // 3) * 0.5, stages=stages,
                         viable=[int(x) for x in viable[r]]))
    sess = P.SchedSession(dev, nreq, sum(len(v) for v in viable) + 1)
    q = P.Queue(n, [r["id"] for r in reqs], [r["arrival"] for r in reqs],
                [s for r in reqs for s in r["stages"]], [r["viable"] for r in reqs])
    slots = sess.add(q)
    by_slot = {int(s): reqs[i] for i, s in enumerate(slots)}
    E = m
    slots_cap = [int(rng.integers(2, 9)) for _ in range(E)]
    weights = [8.0 / 1.5 ** i for i in range(m)]
    inflight = []
    for rnd in range(25):
        occ = [int(rng.integers(0, c + 1)) for c in slots_cap]
        eng = P.Engines(list(range(E)), slots_cap, occ, weights)
        queue_slots = [s for s in sorted(by_slot, key=lambda s: (by_slot[s]["arrival"], by_slot[s]["id"]))
                       if READY in by_slot[s]["stages"]]
        qreqs = [by_slot[s] for s in queue_slots]
        want = _oracle_round(n, m, depth, decl, qreqs, eng, width)
        got = sess.round(eng, width)
        assert [list(t) for t in got.triples] == [list(t) for t in want["triples"]], rnd
        assert got.occupancy == want["occupancy"]
        assert got.utilization == want["utilization"] and got.flexibility == want["flexibility"]
        assert got.skips == want["skips"] and got.states_explored == want["states_explored"]
        assert [queue_slots[t[0]] for t in got.triples] == got.slots
        # apply everything (the round respected capacity), prune the mirror
        sess.dispatch(got)
        for (qi, rid, a, mdl), s in zip(got.triples, got.slots):
            r = by_slot[s]
            r["stages"][a] = 2
            r["viable"] = [int(x) for x in O.prefix_prune(n, m, r["viable"], a, mdl)]
            inflight.append((s, a))
        # complete a random half of the in-flight stages
        rng.shuffle(inflight)
        keep = []
        for k, (s, a) in enumerate(inflight):
            if k % 2 == 0:
                sess.complete(s, a)
                st = by_slot[s]["stages"]
                st[a] = 3
                for b in range(n):
                    if st[b] == 0 and all(st[p] == 3 for p in range(n) if (pred_mask[b] >> p) & 1):
                        st[b] = 1
            else:
                keep.append((s, a))
        inflight = keep
        for s in list(by_slot)[:50]:
            assert sess.viable(s).tolist() == by_slot[s]["viable"]


def _tie_case(rng, n, m, edges, nreq, weights, slots_cap):
    sp = P.ConfigSpace(n, edges, [1.0 + i for i in range(m)], [8.0 / 1.5 ** i for i in range(m)])
    pred_mask = [sum(1 << a for a, b in edges if b == x) for x in range(n)]
    reqs = []
    for r in range(nreq):
        stages = [1 if pred_mask[a] == 0 else 0 for a in range(n)]
        k = int(rng.integers(1, min(sp.size, 12) + 1))
        viable = sorted(set(int(x) for x in rng.integers(0, sp.size, size=k)))
        reqs.append(dict(id=int(500 + r), arrival=float(rng.integers(0, 5)), stages=stages, viable=viable))
    occ = [int(rng.integers(0, c + 1)) for c in slots_cap]
    eng = P.Engines(list(range(m)), slots_cap, occ, weights)
    return sp, reqs, eng


@pytest.mark.parametrize("walker", ["auto", "general"])
def test_beam_ties_match_oracle(walker, monkeypatch):
    """Equal and near-equal engine weights (utilization ties inside one
    parent's children and across parents, decided by flexibility, skips and
    triples_less), widths 1-4 (the fast walker) and 6 (the general one),
    chains and diamonds, against the C oracle."""
    if walker == "general":
        monkeypatch.setenv("AG_SCHED_WALKER", "general")
    rng = np.random.default_rng(11)
    weight_sets = [[1.0, 1.0, 1.0], [2.0, 1.0, 1.0, 0.5], [0.1, 0.2, 0.3, 0.3, 0.1],
                   [1.0, 1.0 + 2 ** -52, 1.0, 0.5], [3.0, 3.0, 3.0, 3.0, 3.0, 3.0, 3.0, 3.0]]
    devs = {}
    for case in range(60):
        ws = weight_sets[case % len(weight_sets)]
        m = len(ws)
        if case % 3 == 2:
            n, edges = 4, DIAMOND
        else:
            n, edges = 3, [(0, 1), (1, 2)]
        cap = [int(rng.integers(1, 4)) for _ in range(m)]
        sp, reqs, eng = _tie_case(rng, n, m, edges, int(rng.integers(3, 25)), ws, cap)
        key = (n, m, len(edges))
        if key not in devs:
            devs[key] = P.Device(sp)
        dev = devs[key]
        q = P.Queue(n, [r["id"] for r in reqs], [r["arrival"] for r in reqs],
                    [s for r in reqs for s in r["stages"]], [r["viable"] for r in reqs])
        order = sorted(range(len(reqs)), key=lambda i: (reqs[i]["arrival"], reqs[i]["id"]))
        for width in (1, 2, 3, 4, 6):
            want = _oracle_round(n, m, sp.depth.tolist(), sp.decl.tolist(), reqs, eng, width)
            got = P.beam_schedule(dev, q, eng, width)
            assert [list(t) for t in got.triples] == [list(t) for t in want["triples"]], (case, width)
            assert got.occupancy == want["occupancy"], (case, width)
            assert got.utilization == want["utilization"] and got.flexibility == want["flexibility"]
            assert got.skips == want["skips"] and got.states_explored == want["states_explored"]
        del order
