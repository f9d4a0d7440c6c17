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


def test_golden_audits(golden):
    """audit_round_fairness on the GPU (stateless: the queue in container
    order, ag_audit_round_fairness) against the reference's violations for
    doctored width-4 assignments and zero for every beam output
    (tests/golden/rounds.json, written by the unmodified reference)."""
    cache = {}
    n = 0
    for j in golden("rounds.json"):
        nn, m = j["n"], j["m"]
        key = (nn, m, tuple(j["graph"]["depth"]))
        if key not in cache:
            sp = P.ConfigSpace(nn, _edges_for(nn, j["graph"]["depth"]), [1.0 + i for i in range(m)],
                               [8.0 / 1.5 ** i for i in range(m)])
            cache[key] = P.Device(sp)
        dev = cache[key]
        reqs, engs = j["requests"], j["engines"]
        q = P.Queue(nn, [r["id"] for r in reqs], [r["arrival"] for r in reqs],
                    [s for r in reqs for s in r["stages"]], [r["viable"] for r in reqs])
        e = P.Engines([x["model"] for x in engs], [x["slots"] for x in engs],
                      [x["occupancy"] for x in engs], [x["weight"] for x in engs])
        for w, want in j["beam"].items():
            assert len(P.audit_round_fairness(dev, q, e, [tuple(t) for t in want["triples"]])) == \
                want["fairness_violations"]
        for d in j["audit"]:
            got = P.audit_round_fairness(dev, q, e, [tuple(t) for t in d["triples"]])
            assert [list(v) for v in got] == d["violations"]
            # right after a stateless round on the same queue the audit reuses
            # the queue already on the device
            P.beam_schedule(dev, q, e, 4)
            got = P.audit_round_fairness(dev, q, e, [tuple(t) for t in d["triples"]])
            assert [list(v) for v in got] == d["violations"]
            n += 1
    assert n >= 120


def test_reference_audit_and_apply_cases():
    """scheduler_test.cpp:211-229 (the audit flags a dropped assignment) and
    :232-265 (apply drops stale triples, a fresh round routes around the full
    pool) on a resident session."""
    sp = P.ConfigSpace.chain(1, 2, [1.0, 2.0], [2.0, 1.0])
    dev = P.Device(sp)
    sess = P.SchedSession(dev, 4, 16)
    q = P.Queue(1, [1, 2], [0.0, 1.0], [READY, READY], [[0, 1], [0, 1]])
    sess.add(q)
    eng = _eng([0, 1], [2, 2], [2.0, 1.0])
    out = sess.round(eng, 4)
    assert len(out.triples) == 2
    assert sess.audit(eng, out.triples) == []
    viol = sess.audit(eng, out.triples[1:])
    assert len(viol) == 1 and viol[0][0] == 1
    # apply with the heavy pool filled between decision and apply
    sp2 = P.ConfigSpace.chain(2, 2, [1.0, 2.0], [2.0, 1.0])
    dev2 = P.Device(sp2)
    s2 = P.SchedSession(dev2, 4, 16)
    q2 = P.Queue(2, [1, 2], [0.0, 1.0], [READY, 0, READY, 0], [[0, 1, 2, 3], [0, 1, 2, 3]])
    s2.add(q2)
    e0 = _eng([0, 1], [2, 2], [2.0, 1.0])
    a = s2.round(e0, 4)
    assert len(a.triples) == 2
    full = _eng([0, 1], [2, 2], [2.0, 1.0], occ=[2, 0])
    flags, na, ns = s2.apply(full, a)
    assert na == 0 and ns == 2 and flags == [False, False]
    assert all(t[3] == 0 for t in a.triples)
    retry = s2.round(full, 4)
    flags, na, ns = s2.apply(full, retry)
    assert ns == 0 and na == 2
    assert all(t[3] == 1 for t in retry.triples)
    # applied stages left the ready set: the next round has nothing to place
    assert s2.round(_eng([0, 1], [2, 2], [2.0, 1.0]), 4).triples == []


@pytest.mark.parametrize("seed", [1, 2])
def test_session_audit_and_apply_match_oracle(seed):
    """Resident-session rounds (chain 5 x 8, predictor sets): the audit of
    doctored assignments against the C oracle's audit_round_fairness, and
    apply_assignment's stale rule against a host replay, round after round."""
    rng = np.random.default_rng(seed)
    n, m, nreq = 5, 8, 600
    sp = P.ConfigSpace.chain(n, m)
    dev = P.Device(sp)
    batch = P.AccuracyBatch.generate(sp, P.GenParams(), nreq, seed)
    pred = P.ConfigPredictor(dev)
    pr = pred.predict_batch(batch.to_device(), P.OracleRouter(0.001))
    torch.cuda.synchronize()
    nv = pr.n_viable.cpu().numpy()
    vv = pr.viable.cpu().numpy().view(np.uint32)
    reqs = [dict(id=int(r), arrival=float(r // 2), stages=[READY] + [0] * (n - 1),
                 viable=[int(x) for x in vv[r, : nv[r]]]) for r in range(nreq)]
    sess = P.SchedSession(dev, nreq, sum(len(r["viable"]) for r in reqs) + 1)
    slots = sess.add(P.Queue(n, [r["id"] for r in reqs], [r["arrival"] for r in reqs],
                             [s for r in reqs for s in r["stages"]], [r["viable"] for r in reqs]))
    by_slot = {int(s): reqs[i] for i, s in enumerate(slots)}
    weights = [8.0 / 1.5 ** i for i in range(m)]
    for rnd in range(6):
        caps = [int(rng.integers(2, 6)) for _ in range(m)]
        occ = [int(rng.integers(0, c + 1)) for c in caps]
        eng = P.Engines(list(range(m)), caps, occ, weights)
        a = sess.round(eng, 4)
        queue_slots = [s for s in sorted(by_slot, key=lambda s: (by_slot[s]["arrival"], by_slot[s]["id"]))
                       if READY in by_slot[s]["stages"]]
        qr = [by_slot[s] for s in queue_slots]
        qd = O.QueueData(n, m, sp.depth.tolist(), sp.decl.tolist(), [r["id"] for r in qr],
                         [r["arrival"] for r in qr], [s for r in qr for s in r["stages"]],
                         [r["viable"] for r in qr], eng.model, eng.slots, eng.occupancy, eng.weight)
        T = len(a.triples)
        docs = [a.triples, a.triples[1:], a.triples[: T // 2], []]
        if T >= 2:
            docs.append([a.triples[1], a.triples[0]] + a.triples[2:])
        for d in docs:
            assert sess.audit(eng, d) == O.audit_round_fairness(qd, d)
        # apply against pools that lost some free slots since the decision
        later = [min(c, o + int(rng.integers(0, 2))) for c, o in zip(caps, occ)]
        leng = P.Engines(list(range(m)), caps, later, weights)
        flags, na, ns = sess.apply(leng, a)
        left = [c - o for c, o in zip(caps, later)]
        want = []
        for t in a.triples:
            ok = left[t[3]] > 0
            left[t[3]] -= ok
            want.append(ok)
        assert flags == want and na == sum(want) and ns == T - sum(want)
        for (qi, rid, ag, mdl), s, ok in zip(a.triples, a.slots, flags):
            if ok:
                r = by_slot[s]
                r["stages"][ag] = 2
                r["viable"] = [int(x) for x in O.prefix_prune(n, m, r["viable"], ag, mdl)]
                sess.complete(s, ag)
                r["stages"][ag] = 3
                if ag + 1 < n:
                    r["stages"][ag + 1] = READY
        for s in list(by_slot)[:40]:
            assert sess.viable(s).tolist() == by_slot[s]["viable"]


def test_session_pool_is_a_capacity():
    """max_configs bounds the viable lists resident at once, not every list
    the session ever adds: continuous add / dispatch (prefix prune) / remove
    cycles through a pool ~4x smaller than the total added, with the live
    lists packed on the device when an add does not fit."""
    rng = np.random.default_rng(7)
    n, m = 3, 4
    sp = P.ConfigSpace.chain(n, m)
    dev = P.Device(sp)
    sess = P.SchedSession(dev, 40, 600)
    mirror = {}
    next_id = 0
    added = 0
    for it in range(40):
        k = 8
        reqs = []
        for _ in range(k):
            v = sorted(set(int(x) for x in rng.integers(0, sp.size, int(rng.integers(5, 25)))))
            reqs.append(dict(id=next_id, arrival=float(next_id), stages=[READY, 0, 0], viable=v))
            next_id += 1
        added += sum(len(r["viable"]) for r in reqs)
        slots = sess.add(P.Queue(n, [r["id"] for r in reqs], [r["arrival"] for r in reqs],
                                 [s for r in reqs for s in r["stages"]], [r["viable"] for r in reqs]))
        for s, r in zip(slots, reqs):
            mirror[int(s)] = r
        # prune some of them in place (agent 0, a candidate model)
        trip, tslots = [], []
        for s in list(mirror)[-k:]:
            r = mirror[s]
            mdl = int((r["viable"][0] // m ** (n - 1)) % m)
            trip.append((0, r["id"], 0, mdl))
            tslots.append(s)
            r["viable"] = [int(x) for x in O.prefix_prune(n, m, r["viable"], 0, mdl)]
            r["stages"][0] = 2
        sess.dispatch(P.Assignment(trip, [], 0.0, 0.0, 0, 0, tslots))
        # the oldest leave
        old = sorted(mirror)[:k] if len(mirror) > 24 else []
        old = sorted(mirror, key=lambda s: mirror[s]["id"])[:k] if len(mirror) > 24 else []
        if old:
            sess.remove(old)
            for s in old:
                del mirror[s]
        for s, r in mirror.items():
            assert sess.viable(s).tolist() == r["viable"], (it, s)
    assert added > 4 * 600


@pytest.mark.parametrize("k", [40, 300])
def test_dispatch_small_and_large_batches_match_oracle(k):
    """ag_sched_dispatch carries small batches in the prune kernel's parameter
    block and stages large ones (more than 768 words of slot / range /
    agent-model data) through pinned memory: both prune every dispatched
    request's viable list exactly as Request::mark_dispatched's prefix prune
    (request.cpp:70-86)."""
    rng = np.random.default_rng(k)
    n, m = 3, 4
    sp = P.ConfigSpace.chain(n, m)
    dev = P.Device(sp)
    sess = P.SchedSession(dev, k, k * 40)
    reqs = []
    for i in range(k):
        v = sorted(set(int(x) for x in rng.integers(0, sp.size, int(rng.integers(5, 30)))))
        reqs.append(dict(id=i, arrival=float(i), stages=[READY, 0, 0], viable=v))
    slots = sess.add(P.Queue(n, [r["id"] for r in reqs], [r["arrival"] for r in reqs],
                             [s for r in reqs for s in r["stages"]], [r["viable"] for r in reqs]))
    trip, tslots = [], []
    for s, r in zip(slots, reqs):
        mdl = int((r["viable"][int(rng.integers(0, len(r["viable"])))] // m ** (n - 1)) % m)
        trip.append((0, r["id"], 0, mdl))
        tslots.append(int(s))
        r["viable"] = [int(x) for x in O.prefix_prune(n, m, r["viable"], 0, mdl)]
    sess.dispatch(P.Assignment(trip, [], 0.0, 0.0, 0, 0, tslots))
    for s, r in zip(slots, reqs):
        assert sess.viable(int(s)).tolist() == r["viable"]
