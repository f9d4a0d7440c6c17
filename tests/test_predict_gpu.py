"""Chain-mode routing parity: ConfigPredictor::predict on the GPU against the
reference's golden predictions (tests/golden/predict.json, chains.json) and
the C oracle restatement at larger sizes.  Bit-exact: viable sets, search and
verify evaluation counts, router_time (fp64, identical) and truncated."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

INF = math.inf


def _space_with_cost(n, m, cost):
    return P.ConfigSpace(n, [(i - 1, i) for i in range(1, n)], cost,
                         [8.0 / 1.5 ** i for i in range(m)])


def test_chain_plans_match_reference(golden):
    for c in golden("chains.json"):
        space = P.ConfigSpace.chain(c["n"], c["m"])
        dev = P.Device(space)
        pred = P.ConfigPredictor(dev, c["cap"], c["limit"])
        assert pred.exhaustive == c["exhaustive"]
        assert pred.chains().tolist() == c["chains"]


def _check_batch(res, wants):
    nv = res.n_viable.cpu().numpy()
    viable = res.viable.cpu().numpy()
    se, ve = res.search_evals.cpu().numpy(), res.verify_evals.cpu().numpy()
    rt, tr = res.router_time.cpu().numpy(), res.truncated.cpu().numpy()
    for i, w in enumerate(wants):
        assert viable[i, : nv[i]].tolist() == list(w["viable"]), i
        assert se[i] == w["search_evals"], i
        assert ve[i] == w["verify_evals"], i
        assert rt[i] == w["router_time"], i
        assert bool(tr[i]) == bool(w["truncated"]), i


def test_golden_predictions(golden):
    for case in golden("predict.json"):
        n, m = case["n"], case["m"]
        space = _space_with_cost(n, m, case["cost"])
        dev = P.Device(space)
        pred = P.ConfigPredictor(dev)
        reqs = case["requests"]
        batch = P.AccuracyBatch.from_lists(n, [r["seeds"] for r in reqs],
                                           [r["removed"] for r in reqs], [r["id"] for r in reqs])
        router = (P.NoisyRouter(case["fp"], case["fn"], case["noise_seed"], case["latency"])
                  if case["noisy"] else P.OracleRouter(case["latency"]))
        budget = INF if case["budget"] < 0 else case["budget"]
        res = pred.predict_batch(batch.to_device(), router, budget)
        torch.cuda.synchronize()
        _check_batch(res, reqs)


@pytest.mark.parametrize("n,m,R,noisy,latency,budget", [
    (5, 8, 2000, False, 0.002, INF), (5, 8, 500, True, 0.002, INF),
    (5, 8, 500, False, 0.002, 0.03), (5, 8, 300, True, 0.001, 0.02),
    (3, 4, 800, True, 0.002, 0.05), (4, 3, 800, False, 0.002, 0.01),
    (8, 12, 64, True, 0.002, INF), (6, 4, 200, False, 0.0015, 0.04),
    (2, 2, 50, False, 1.0, 1.0), (1, 3, 30, True, 0.5, 0.7)])
def test_predict_matches_oracle(n, m, R, noisy, latency, budget):
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space)
    pred = P.ConfigPredictor(dev)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=11 + n)
    router = P.NoisyRouter(0.05, 0.3, 77, latency) if noisy else P.OracleRouter(latency)
    # per-request budgets around the given one exercise truncation points
    rng = np.random.default_rng(n * 100 + m)
    budgets = (np.full(R, budget) if math.isinf(budget) else
               budget * rng.uniform(0.0, 2.0, R)).astype(np.float64)
    res = pred.predict_batch(batch.to_device(), router, torch.from_numpy(budgets).cuda())
    torch.cuda.synchronize()
    tb = O.TruthBatch(n, m, [batch.seeds_of(r) for r in range(R)],
                      [batch.removed_of(r) for r in range(R)], batch.request_ids)
    orouter = O.Router(router.kind, router.fp, router.fn, router.noise_seed, latency)
    chains = pred.chains()
    wants = [O.predict(tb, orouter, space.cost, chains, r, float(budgets[r])) for r in range(R)]
    _check_batch(res, wants)


def test_predict_violations_and_zero_budget():
    space = P.ConfigSpace.chain(3, 4)
    dev = P.Device(space)
    pred = P.ConfigPredictor(dev)
    batch = P.AccuracyBatch.generate(space, P.GenParams(violation_rate=0.05), 200, seed=4)
    res = pred.predict_batch(batch.to_device(), P.OracleRouter(0.002), 0.0)
    torch.cuda.synchronize()
    assert (res.n_viable.cpu() == 1).all()  # zero budget -> {top} (predictor_test.cpp:196-213)
    assert (res.search_evals.cpu() == 0).all() and (res.truncated.cpu() == 1).all()
    assert (res.viable[:, 0].cpu() == space.top).all()
    tb = O.TruthBatch(3, 4, [batch.seeds_of(r) for r in range(200)],
                      [batch.removed_of(r) for r in range(200)], batch.request_ids)
    res = pred.predict_batch(batch.to_device(), P.OracleRouter(0.002), INF)
    torch.cuda.synchronize()
    chains = pred.chains()
    wants = [O.predict(tb, O.Router(0, 0, 0, 0, 0.002), space.cost, chains, r, INF)
             for r in range(200)]
    _check_batch(res, wants)
