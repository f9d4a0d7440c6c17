"""Accurate-set trace writer (ag_trace_write) on the GPU: for
spaces below, at and above the 4096-configuration bitmap limit, every
record decodes to the oracle's accurate set (AccurateSet::contains over the
canonical enumeration, accuracy.cpp:116-124), ids and arrivals round-trip
exactly, and an unwritable path fails with AG_ERR_IO."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2511_20975_b200 import trace as T  # noqa: E402


@pytest.mark.parametrize("n,m,R,enc", [(3, 4, 200, "bitmap"), (4, 8, 60, "bitmap"), (6, 4, 60, "bitmap"),
                                       (5, 8, 40, "list"), (2, 2, 30, "bitmap")])
def test_trace_round_trip_matches_oracle(tmp_path, n, m, R, enc):
    sp = P.ConfigSpace.chain(n, m)
    dev = P.Device(sp)
    batch = P.AccuracyBatch.generate(sp, P.GenParams(violation_rate=0.05 if sp.size <= 4096 else 0.0), R,
                                     seed=n * 10 + m,
                                     first_id=1000)
    arrival = np.cumsum(np.random.default_rng(1).exponential(0.37, R))
    path = tmp_path / "trace.jsonl"
    nbytes = T.write_trace(dev, batch, str(path), arrival)
    assert nbytes == path.stat().st_size
    text = path.read_text().splitlines()
    assert len(text) == R and all(f'"encoding": "{enc}"' in ln for ln in text)
    ids, arr, offs, mem = T.read_trace(str(path))
    assert ids.tolist() == batch.request_ids.tolist()
    assert arr.tolist() == arrival.tolist()
    tb = O.TruthBatch(n, m, [batch.seeds_of(r) for r in range(R)], [batch.removed_of(r) for r in range(R)],
                      batch.request_ids)
    for r in range(R):
        cnt, words = O.enumerate_bitmap(tb, O.Router(0, 0, 0, 0, 0), r, 0, sp.size)
        want = np.nonzero(np.unpackbits(words.view(np.uint8), bitorder="little"))[0][:cnt]
        assert mem[offs[r]:offs[r + 1]].tolist() == want.tolist(), r


def test_trace_unwritable_path_is_io_error(tmp_path):
    sp = P.ConfigSpace.chain(3, 3)
    dev = P.Device(sp)
    batch = P.AccuracyBatch.generate(sp, P.GenParams(), 4, seed=1)
    with pytest.raises(P.AgError) as e:
        T.write_trace(dev, batch, str(tmp_path / "no_such_dir" / "t.jsonl"))
    assert e.value.code == 3  # AG_ERR_IO (errors.h IoError)
