"""Trace I/O of accurate-configuration sets (SURVEY.md §8(f)
rank 4): the line-delimited trace of request id, arrival and accurate set --
a bitmap over the canonical enumeration for M^N <= 4096, an explicit member
list otherwise.  Writing enumerates the sets on the device
(ag_trace_write); reading decodes either encoding into a member CSR that the
scheduler (viable sets) and the runtime-cost argmin (select_per_input)
take directly."""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from ._capi import check, lib
from .routing import AccuracyBatch, Device, _ptr


def write_trace(device: Device, batch: AccuracyBatch, path: str, arrival=None) -> int:
    """ag_trace_write: one line per request of `batch`; returns bytes written."""
    arr = None if arrival is None else np.ascontiguousarray(arrival, np.float64)
    n = C.c_uint64()
    t = batch.c_struct()
    check(lib().ag_trace_write(device.handle, C.byref(t), C.c_void_p(_ptr(arr)),
                               str(path).encode(), C.byref(n)))
    return n.value


def decode_set(acc: dict) -> np.ndarray:
    """Ascending canonical indices of one record's accurate set."""
    if acc["encoding"] == "bitmap":
        raw = np.frombuffer(bytes.fromhex(acc["bits"]), np.uint8)
        bits = np.unpackbits(raw, bitorder="little")[: int(acc["size"])]
        return np.nonzero(bits)[0].astype(np.uint32)
    if acc["encoding"] == "list":
        return np.asarray(acc["members"], np.uint32)
    raise ValueError(f"unknown accurate-set encoding {acc['encoding']!r}")


def read_trace(path: str):
    """(ids u64 [R], arrival f64 [R], offsets i64 [R+1], members u32 [total])."""
    ids, arr, sets = [], [], []
    with open(path) as f:
        for line in f:
            if not line.strip():
                continue
            rec = json.loads(line)
            ids.append(int(rec["id"]))
            arr.append(float(rec["arrival"]))
            sets.append(decode_set(rec["accurate"]))
    offsets = np.zeros(len(sets) + 1, np.int64)
    for i, s in enumerate(sets):
        offsets[i + 1] = offsets[i] + len(s)
    members = np.concatenate(sets) if sets and offsets[-1] else np.zeros(0, np.uint32)
    return np.asarray(ids, np.uint64), np.asarray(arr, np.float64), offsets, members
