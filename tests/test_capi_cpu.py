"""CPU-only checks of the product library: it loads, exports every symbol the
public header declares, and its host-side pieces (space construction, input
generator) agree with the reference's golden vectors."""
import ctypes as C

import numpy as np
import pytest

import paper_2511_20975_b200 as P
from paper_2511_20975_b200 import _capi


def test_library_exports_every_header_symbol():
    L = P.lib()
    syms = _capi.header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s


def test_space_matches_reference_graphs(golden):
    for g in golden("graph.json"):
        n = g["n"]
        sp = P.ConfigSpace(n, g["edges"], [1.0 + i for i in range(3)], [3.0, 2.0, 1.0])
        assert sp.decl.tolist() == g["decl"]
        assert sp.depth.tolist() == g["depth"]
        assert sp.size == 3 ** n


def test_space_validation():
    with pytest.raises(P.ValidationError):
        P.ConfigSpace(2, [(0, 1), (1, 0)], [1, 2], [2, 1])  # cycle
    with pytest.raises(P.ValidationError):
        P.ConfigSpace(2, [(0, 0)], [1, 2], [2, 1])  # self loop
    with pytest.raises(P.ValidationError):
        P.ConfigSpace(2, [(0, 5)], [1, 2], [2, 1])  # unknown endpoint
    with pytest.raises(P.ValidationError):
        P.ConfigSpace(1, [], [1, 1], [2, 1])  # cost not strictly increasing
    with pytest.raises(P.ValidationError):
        P.ConfigSpace(1, [], [1, 2], [1, 2])  # throughput not strictly decreasing
    with pytest.raises(P.ValidationError):
        P.ConfigSpace(1, [], [1], [1])  # < 2 tiers


def test_generator_matches_reference(golden):
    rows = golden("truth.json")
    groups = {}
    for r in rows:
        groups.setdefault((r["n"], r["m"], tuple(r["params"]), r["seed"]), []).append(r)
    for (n, m, params, seed), rs in groups.items():
        sp = P.ConfigSpace.chain(n, m)
        ids = [r["id"] for r in rs]
        assert ids == list(range(len(ids)))
        b = P.AccuracyBatch.generate(sp, P.GenParams(*params), len(rs), seed)
        for i, r in enumerate(rs):
            assert b.seeds_of(i).tolist() == r["seeds"], (n, m, params, seed, i)
            assert b.removed_of(i).tolist() == r["removed"]


def test_generator_validation():
    sp = P.ConfigSpace.chain(7, 4)  # 16384 > 4096
    with pytest.raises(P.ValidationError):
        P.AccuracyBatch.generate(sp, P.GenParams(violation_rate=0.1), 4, 1)
    with pytest.raises(P.ValidationError):
        P.AccuracyBatch.generate(sp, P.GenParams(p_easy=-1), 4, 1)


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    sp = P.ConfigSpace.chain(2, 2)
    h = C.c_void_p()
    rc = P.lib().ag_ctx_create(sp.handle, 0, C.byref(h))
    assert rc == _capi.AG_ERR_CUDA
