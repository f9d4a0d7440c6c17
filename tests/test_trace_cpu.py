"""Trace reader (SPEC.md:475 accurate-set trace, paper_2511_20975_b200.trace)
on hand-written records of both encodings: the bitmap over the canonical
enumeration (byte k = indices 8k..8k+7, bit 0 first) and the explicit list."""
import json

import numpy as np

from paper_2511_20975_b200 import trace as T


def test_read_both_encodings(tmp_path):
    p = tmp_path / "t.jsonl"
    recs = [{"id": 7, "arrival": 0.5, "accurate": {"encoding": "bitmap", "size": 12, "bits": "a50f"}},
            {"id": 9, "arrival": 1.25, "accurate": {"encoding": "list", "size": 5000, "members": [3, 4999]}},
            {"id": 11, "arrival": 2.0, "accurate": {"encoding": "bitmap", "size": 3, "bits": "00"}}]
    p.write_text("".join(json.dumps(r) + "\n" for r in recs))
    ids, arr, offs, mem = T.read_trace(str(p))
    assert ids.tolist() == [7, 9, 11] and arr.tolist() == [0.5, 1.25, 2.0]
    assert offs.tolist() == [0, 8, 10, 10]
    assert mem.tolist() == [0, 2, 5, 7, 8, 9, 10, 11, 3, 4999]
    # bits beyond `size` are ignored
    assert T.decode_set({"encoding": "bitmap", "size": 4, "bits": "ff"}).tolist() == [0, 1, 2, 3]
