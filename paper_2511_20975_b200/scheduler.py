"""Per-stage scheduler: host mirror of beam_schedule / Request over the C ABI.

Reference: include/aragog/scheduler.h:37-118, src/scheduler.cpp:29-454,
include/aragog/request.h:30-67.  `beam_schedule` is the stateless drop-in
(uploads the queue every call); `SchedSession` keeps the in-flight requests
resident in HBM across rounds, as the simulator's event loop uses them.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import check, lib
from .routing import Device, _ptr

PENDING, READY, INFLIGHT, DONE = 0, 1, 2, 3


class CEngines(C.Structure):
    _fields_ = [("n_engines", C.c_int32), ("model", C.c_void_p), ("slots", C.c_void_p),
                ("occupancy", C.c_void_p), ("weight", C.c_void_p)]


class CTriple(C.Structure):
    _fields_ = [("request_index", C.c_int32), ("agent", C.c_int32), ("model", C.c_int32),
                ("slot", C.c_int32), ("request_id", C.c_uint64)]


class CAssignment(C.Structure):
    _fields_ = [("n_triples", C.c_int32), ("pad", C.c_int32), ("utilization", C.c_double),
                ("flexibility", C.c_double), ("skips", C.c_int64), ("states_explored", C.c_uint64)]


class CQueue(C.Structure):
    _fields_ = [("n_requests", C.c_int32), ("ids", C.c_void_p), ("arrival", C.c_void_p),
                ("stages", C.c_void_p), ("viable_ptr", C.c_void_p), ("viable", C.c_void_p)]


@dataclass
class Engines:
    """vector<EngineState> (engine.h:38-53): one pool per tier."""
    model: list
    slots: list
    occupancy: list
    weight: list

    def c(self):
        self._arrs = [np.ascontiguousarray(self.model, np.int32),
                      np.ascontiguousarray(self.slots, np.int32),
                      np.ascontiguousarray(self.occupancy, np.int32),
                      np.ascontiguousarray(self.weight, np.float64)]
        return CEngines(len(self.model), *[_ptr(a) for a in self._arrs])


@dataclass
class Assignment:
    """Assignment (scheduler.h:76-83); triples are (request_index, request_id,
    agent, model) as in the reference, `slots` the session slots."""
    triples: list
    occupancy: list
    utilization: float
    flexibility: float
    skips: int
    states_explored: int
    slots: list = field(default_factory=list)


class Queue:
    """The round's vector<const Request*> as flat host arrays."""

    def __init__(self, n_agents, ids, arrival, stages, viable_lists):
        self.n = n_agents
        self.ids = np.ascontiguousarray(ids, np.uint64)
        self.arrival = np.ascontiguousarray(arrival, np.float64)
        self.stages = np.ascontiguousarray(np.asarray(stages, np.uint8).reshape(-1))
        ptr = [0]
        for v in viable_lists:
            ptr.append(ptr[-1] + len(v))
        self.viable_ptr = np.asarray(ptr, np.int64)
        self.viable = np.ascontiguousarray(
            np.concatenate([np.asarray(v, np.uint32) for v in viable_lists]) if ptr[-1] else
            np.zeros(1, np.uint32))

    def c(self):
        return CQueue(len(self.ids), _ptr(self.ids), _ptr(self.arrival), _ptr(self.stages),
                      _ptr(self.viable_ptr), _ptr(self.viable))


def _unpack(res: CAssignment, trip, occ, E):
    tr = [(trip[i].request_index, trip[i].request_id, trip[i].agent, trip[i].model)
          for i in range(res.n_triples)]
    return Assignment(tr, list(occ[:E]), res.utilization, res.flexibility, res.skips,
                      res.states_explored, [trip[i].slot for i in range(res.n_triples)])


def beam_schedule(device: Device, queue: Queue, engines: Engines, beam_width: int = 4) -> Assignment:
    """beam_schedule(queue, engines, {beam_width}) (scheduler.cpp:289-378)."""
    cap = max(1, int(sum(max(0, s - o) for s, o in zip(engines.slots, engines.occupancy))) + 1)
    trip = (CTriple * cap)()
    occ = np.zeros(max(1, len(engines.model)), np.int32)
    res = CAssignment()
    q, e = queue.c(), engines.c()
    check(lib().ag_beam_schedule(device.handle, C.byref(q), C.byref(e), beam_width,
                                 C.byref(res), trip, cap, C.c_void_p(_ptr(occ))))
    return _unpack(res, trip, occ, len(engines.model))


def _ctriples(triples, slots):
    arr = (CTriple * max(1, len(triples)))()
    for k, ((qi, rid, a, m), sl) in enumerate(zip(triples, slots)):
        arr[k] = CTriple(qi, a, m, sl, rid)
    return arr


def _audit(call, engines: Engines, triples) -> list:
    n = len(triples)
    arr = _ctriples(triples, [-1] * n)
    cap = 4096
    ids = np.zeros(cap, np.uint64)
    ags = np.zeros(cap, np.int32)
    nv = C.c_int32()
    e = engines.c()
    check(call(C.byref(e), n, arr, C.c_void_p(_ptr(ids)), C.c_void_p(_ptr(ags)), cap, C.byref(nv)))
    return [(int(ids[i]), int(ags[i])) for i in range(min(nv.value, cap))]


def audit_round_fairness(device: Device, queue: Queue, engines: Engines, triples) -> list:
    """audit_round_fairness(queue, engines, assignment) (scheduler.cpp:456-480),
    stateless: request_index is the container index of `queue`."""
    q = queue.c()
    return _audit(lambda *a: lib().ag_audit_round_fairness(device.handle, C.byref(q), *a), engines, triples)


class SchedSession:
    """Resident requests (ag_sched): add -> round -> dispatch -> complete."""

    def __init__(self, device: Device, max_requests: int, max_configs: int):
        self.device = device
        h = C.c_void_p()
        check(lib().ag_sched_create(device.handle, max_requests, C.c_uint64(max_configs), C.byref(h)))
        self._h = h
        self._trip = None

    def add(self, queue: Queue) -> np.ndarray:
        """Request::make for each row; returns their slots."""
        slots = np.zeros(max(1, len(queue.ids)), np.int32)
        q = queue.c()
        check(lib().ag_sched_add(self._h, C.byref(q), C.c_void_p(_ptr(slots))))
        return slots[: len(queue.ids)]

    def remove(self, slots):
        s = np.ascontiguousarray(slots, np.int32)
        check(lib().ag_sched_remove(self._h, len(s), C.c_void_p(_ptr(s))))

    def complete(self, slot: int, agent: int):
        """Request::mark_complete (request.cpp:88-107)."""
        check(lib().ag_sched_complete(self._h, int(slot), int(agent)))

    def round(self, engines: Engines, beam_width: int = 4) -> Assignment:
        cap = max(1, int(sum(max(0, s - o) for s, o in zip(engines.slots, engines.occupancy))) + 1)
        if self._trip is None or len(self._trip) < cap:
            self._trip = (CTriple * max(cap, 256))()
        occ = np.zeros(max(1, len(engines.model)), np.int32)
        res = CAssignment()
        e = engines.c()
        check(lib().ag_sched_round(self._h, C.byref(e), beam_width, C.byref(res), self._trip,
                                   len(self._trip), C.c_void_p(_ptr(occ))))
        return _unpack(res, self._trip, occ, len(engines.model))

    def dispatch(self, assignment: Assignment, keep=None):
        """Request::mark_dispatched for the applied triples (default: all)."""
        idx = range(len(assignment.triples)) if keep is None else keep
        arr = (CTriple * max(1, len(idx)))()
        for k, i in enumerate(idx):
            qi, rid, a, m = assignment.triples[i]
            arr[k] = CTriple(qi, a, m, assignment.slots[i], rid)
        check(lib().ag_sched_dispatch(self._h, len(idx), arr))

    def apply(self, engines: Engines, assignment: Assignment):
        """apply_assignment (scheduler.cpp:421-454) on the session: a triple
        whose pool is already full is stale (dropped), the rest dispatch.
        Returns (applied flags, number applied, number stale)."""
        n = len(assignment.triples)
        arr = _ctriples(assignment.triples, assignment.slots or [-1] * n)
        flags = np.zeros(max(1, n), np.uint8)
        na, ns = C.c_int32(), C.c_int32()
        e = engines.c()
        check(lib().ag_sched_apply(self._h, C.byref(e), n, arr, C.c_void_p(_ptr(flags)),
                                   C.byref(na), C.byref(ns)))
        return flags[:n].astype(bool).tolist(), na.value, ns.value

    def audit(self, engines: Engines, triples) -> list:
        """audit_round_fairness (scheduler.cpp:456-480) of an assignment's
        triples (request_index, request_id, agent, model) against the last
        round's queue; returns [(RequestId, agent)] in pair order."""
        return _audit(lambda *a: lib().ag_sched_audit(self._h, *a), engines, triples)

    def round_timing(self):
        """Device phase durations (us) of the last round: setup, first
        candidate chunk, walk, finalize.  Also sets walk_cycles (find, build,
        rank, adopt), walk_counts (steps, children) and chunk_us (the first
        producer chunk: loads, scan, records, histogram rows)."""
        t = np.zeros(16, np.uint64)
        check(lib().ag_sched_round_timing(self._h, C.c_void_p(_ptr(t))))
        self.walk_cycles = t[5:9].astype(np.float64)
        self.walk_counts = t[9:11].astype(np.int64)
        self.ctx_cycles = self.walk_counts
        self.chunk_us = np.diff(np.concatenate([[float(t[1])], t[11:15].astype(np.float64)])) / 1e3
        # producers' end relative to the walk's end (us; > 0: they finished later)
        self.producers_after_walk_us = (float(t[15]) - float(t[3])) / 1e3 if t[15] else 0.0
        return np.diff(t[:5].astype(np.float64)) / 1e3

    def host_timing(self):
        """Host-clock split (us) of the last round call: record preparation,
        launch call, wait for the completion flag, result readback."""
        t = np.zeros(4, np.float64)
        check(lib().ag_sched_round_host_timing(self._h, C.c_void_p(_ptr(t))))
        return t

    def last_round_us(self) -> float:
        """Host wall time of the last round inside the C ABI call."""
        f = lib().ag_sched_last_round_us
        f.restype = C.c_double
        return float(f(self._h))

    def viable(self, slot: int) -> np.ndarray:
        n = C.c_int64()
        check(lib().ag_sched_viable(self._h, int(slot), None, 0, C.byref(n)))
        out = np.zeros(max(1, n.value), np.uint32)
        check(lib().ag_sched_viable(self._h, int(slot), C.c_void_p(_ptr(out)), len(out), C.byref(n)))
        return out[: n.value]

    def __del__(self):
        try:  # module globals may already be gone at interpreter shutdown
            _capi.release("ag_sched_destroy", getattr(self, "_h", None))
        except Exception:  # noqa: BLE001
            pass
        self._h = None


class CLoad(C.Structure):
    _fields_ = [("n_tiers", C.c_int32), ("occupancy", C.c_void_p), ("queued_ahead", C.c_void_p),
                ("slots", C.c_void_p), ("mean", C.c_void_p)]


PER_INPUT_STATIC, PER_INPUT_RUNTIME_COST = 2, 3


@dataclass
class RuntimeCostContext:
    """RuntimeCostContext (workload.h:64-69); mean[m] = ServiceTimeModel::mean."""
    occupancy: list
    queued_ahead: list
    slots: list
    mean: list

    def c(self):
        self._arrs = [np.ascontiguousarray(self.occupancy, np.int32),
                      np.ascontiguousarray(self.queued_ahead, np.int32),
                      np.ascontiguousarray(self.slots, np.int32),
                      np.ascontiguousarray(self.mean, np.float64)]
        return CLoad(len(self.slots), *[_ptr(a) for a in self._arrs])


def select_per_input(device: Device, members, offsets, kind=PER_INPUT_RUNTIME_COST, ctx=None,
                     check_errors=True):
    """select_per_input_config for every request of a member CSR (device
    tensors: members int32 [total], offsets int64 [R+1]).  Returns device
    tensors (chosen canonical index, estimate).  The C call is asynchronous;
    with check_errors the stream is synchronised so that the reference's
    ValidationErrors (an empty set, a tier missing from the load context)
    raise here, as select_per_input_config throws (workload.cpp:140-156)."""
    import torch

    R = offsets.numel() - 1
    chosen = torch.zeros(max(R, 1), dtype=torch.int32, device=device.torch_device)
    est = torch.zeros(max(R, 1), dtype=torch.float64, device=device.torch_device)
    load = ctx.c() if ctx is not None else None
    check(lib().ag_select_per_input(device.handle, C.c_void_p(_ptr(members)), C.c_void_p(_ptr(offsets)),
                                    R, kind, C.byref(load) if load is not None else None,
                                    C.c_void_p(_ptr(chosen)), C.c_void_p(_ptr(est))))
    if check_errors:
        check(lib().ag_ctx_synchronize(device.handle))
    return chosen[:R], est[:R]


def select_bitmap(device: Device, bitmap, counts, begin: int, end: int, kind=PER_INPUT_RUNTIME_COST, ctx=None,
                  check_errors=True, records=None):
    """select_per_input_config straight from an enumerate-mode verdict bitmap
    (device tensors: bitmap int32 [R, W] over [begin, end), counts int64 [R])
    -- ag_select_bitmap: the same (chosen canonical index, estimate) as
    select_per_input over the compacted members, without the member list.
    records: optional int64 [R, 4] device tensor receiving the shard records
    (ag_shard_records' layout; empty sets allowed then)."""
    import torch

    R = counts.numel()
    chosen = torch.zeros(max(R, 1), dtype=torch.int32, device=device.torch_device)
    est = torch.zeros(max(R, 1), dtype=torch.float64, device=device.torch_device)
    load = ctx.c() if ctx is not None else None
    check(lib().ag_select_bitmap(device.handle, C.c_void_p(_ptr(bitmap)), C.c_void_p(_ptr(counts)),
                                 C.c_uint64(begin), C.c_uint64(end), R, kind,
                                 C.byref(load) if load is not None else None, C.c_void_p(_ptr(chosen)),
                                 C.c_void_p(_ptr(est)), C.c_void_p(_ptr(records) if records is not None else None)))
    if check_errors:
        check(lib().ag_ctx_synchronize(device.handle))
    return chosen[:R], est[:R]


def select_per_input_host(device: Device, batch, kind=PER_INPUT_RUNTIME_COST, ctx=None):
    """select_per_input_config for a host AccuracyBatch end to end
    (ag_select_per_input_host: oracle verdict bitmaps over the whole space
    built on the device, re-cost + arg-min straight from them).  Returns
    numpy (chosen canonical index uint32 [R], estimate float64 [R])."""
    R = batch.n_requests
    chosen = np.zeros(max(R, 1), np.uint32)
    est = np.zeros(max(R, 1), np.float64)
    t = batch.c_struct()
    load = ctx.c() if ctx is not None else None
    check(lib().ag_select_per_input_host(device.handle, C.byref(t), kind,
                                         C.byref(load) if load is not None else None,
                                         C.c_void_p(_ptr(chosen)), C.c_void_p(_ptr(est))))
    return chosen[:R], est[:R]


def select_bitmap_stats(device: Device, enable: bool) -> int:
    """ag_select_bitmap_stats: start (enable) or stop counting the words the
    exact pass of select_bitmap evaluates; returns the count on stop."""
    out = C.c_uint64()
    check(lib().ag_select_bitmap_stats(device.handle, 1 if enable else 0, C.byref(out)))
    return int(out.value)


def select_per_workflow(device: Device, sample, tolerance: float = 0.0):
    """select_per_workflow_config(sample, space, tolerance) (workload.cpp:99-127)
    over a host AccuracyBatch, without the 4096-configuration guard: returns
    (canonical index, accurate count over the sample)."""
    chosen = C.c_uint64()
    hits = C.c_uint64()
    t = sample.c_struct()
    check(lib().ag_select_per_workflow_host(device.handle, C.byref(t), C.c_double(tolerance),
                                            C.byref(chosen), C.byref(hits)))
    return int(chosen.value), int(hits.value)


def _queued_ahead(self) -> list:
    """snapshot_load's queued_ahead per model tier (simulation.cpp:194-213)."""
    out = np.zeros(64, np.int32)
    check(lib().ag_sched_queued_ahead(self._h, C.c_void_p(_ptr(out))))
    return out[: self.device.space.m].tolist()


SchedSession.queued_ahead = _queued_ahead
