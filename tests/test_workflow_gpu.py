"""Per-workflow baseline on the GPU (select_per_workflow_config,
workload.cpp:99-127): bit-exact against the
reference's picks (tests/golden/workflow.json) and, beyond the reference's
4096-configuration guard, against the C oracle restatement."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _tb(space, batch):
    return O.TruthBatch(space.n, space.m, [batch.seeds_of(r) for r in range(batch.n_requests)],
                        [batch.removed_of(r) for r in range(batch.n_requests)], batch.request_ids)


def test_matches_reference_picks(golden):
    devs = {}
    for w in golden("workflow.json"):
        key = (w["n"], w["m"])
        if key not in devs:
            sp = P.ConfigSpace.chain(w["n"], w["m"])
            devs[key] = (sp, P.Device(sp))
        sp, dev = devs[key]
        batch = P.AccuracyBatch.generate(sp, P.GenParams(violation_rate=w["violation_rate"]),
                                         w["count"], w["seed"])
        pick, hits = P.select_per_workflow(dev, batch, w["tolerance"])
        assert pick == w["pick"], w
        assert hits >= (1 - w["tolerance"]) * w["count"]


@pytest.mark.parametrize("n,m,R,tol", [(5, 8, 300, 0.0), (5, 8, 300, 0.1), (4, 6, 57, 0.25),
                                       (3, 4, 5000, 0.0), (3, 4, 5000, 0.4)])
def test_large_spaces_and_many_sets(n, m, R, tol):
    """Beyond 4096 configurations (the reference refuses) and beyond one
    2048-row counting chunk (atomic accumulation)."""
    sp = P.ConfigSpace.chain(n, m)
    dev = P.Device(sp)
    batch = P.AccuracyBatch.generate(sp, P.GenParams(), R, seed=77 + R)
    pick, hits = P.select_per_workflow(dev, batch, tol)
    want, want_hits = O.select_per_workflow(n, m, [1.5 ** i for i in range(m)], _tb(sp, batch), tol)
    assert (pick, hits) == (want, want_hits)


def test_validation():
    sp = P.ConfigSpace.chain(3, 3)
    dev = P.Device(sp)
    with pytest.raises(P.ValidationError, match="empty"):
        P.select_per_workflow(dev, P.AccuracyBatch.from_lists(3, [], []), 0.0)
    batch = P.AccuracyBatch.generate(sp, P.GenParams(), 4, seed=1)
    for bad in (-0.1, 1.5, float("nan")):
        with pytest.raises(P.ValidationError, match="tolerance"):
            P.select_per_workflow(dev, batch, bad)
