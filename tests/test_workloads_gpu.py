"""The config-3 scheduling loop through the GPU session makes exactly the
decisions of the unmodified reference loop (oracle/_ref/ref_bench sched):
same decision hash over every round (triples, utilization, explored, skips)."""
import json
import os
import subprocess

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from paper_2511_20975_b200 import workloads as W  # noqa: E402

REF = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "ref_bench")


def test_mix_matches_reference(golden):
    for row in golden("rng.json"):
        a, b, c = row["words"]
        assert W.mix(a, b, c) == row["mix3"]


@pytest.mark.parametrize("inflight,beam,rounds,exhaustive", [(600, 4, 40, 0), (400, 1, 30, 0),
                                                              (200, 4, 25, 1)])
def test_config3_decisions_match_reference(inflight, beam, rounds, exhaustive):
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/ref_bench not built")
    out = subprocess.run([REF, "sched", str(inflight), str(beam), str(rounds), "1", str(exhaustive)],
                         capture_output=True, text=True, check=True).stdout
    ref = json.loads(out.strip().splitlines()[-1])
    dev = P.Device(W.config2_space())
    c3 = W.Config3(dev, inflight=inflight, rounds=rounds, seed=1, beam=beam,
                   exhaustive=bool(exhaustive))
    lat, h, assigned = c3.run()
    assert assigned == ref["assigned"]
    assert f"{h:016x}" == ref["hash"]
