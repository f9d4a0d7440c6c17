"""Synthetic BASELINE workloads, built on the product API.

The generators are pure functions of their seeds, restating the reference's
own input synthesis (rng::mix / splitmix64, include/aragog/rng.h:34-51;
generate_accurate_set, src/accuracy.cpp:144-198, via ag_generate_truth), so
the GPU arm and the reference arm (oracle/ref_bench.cpp) see identical inputs.
"""
from __future__ import annotations

import time

import numpy as np

from .predictor import ConfigPredictor
from .routing import AccuracyBatch, ConfigSpace, Device, GenParams, OracleRouter
from .scheduler import PENDING, READY, DONE, Engines, Queue, SchedSession

MASK = (1 << 64) - 1
GAMMA = 0x9e3779b97f4a7c15


def _splitmix(x):
    z = (x + GAMMA) & MASK
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & MASK
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & MASK
    return z ^ (z >> 31)


def mix(*words):
    """rng::mix (rng.h:43-51)."""
    s = 0x6a09e667f3bcc909
    for w in words:
        s ^= (w + GAMMA + ((s << 6) & MASK) + (s >> 2)) & MASK
        s = _splitmix(s)
    return s


def config2_space():
    """BASELINE config 2: chain of 5 agents x 8 tiers, cost x1.5 / weight /1.5."""
    return ConfigSpace.chain(5, 8)


def config3_engines(rnd, seed, weights, n_pools=8, slots=32):
    """Round rnd's load: all pools full, then F = {1, 8, 64}[mix(seed, rnd) % 3]
    draws e = mix(seed, rnd, j) % 8 free one slot of a non-empty pool."""
    F = (1, 8, 64)[mix(seed, rnd) % 3]
    occ = [slots] * n_pools
    for j in range(F):
        e = mix(seed, rnd, j) % n_pools
        if occ[e] > 0:
            occ[e] -= 1
    return Engines(list(range(n_pools)), [slots] * n_pools, occ, list(weights[:n_pools])), F


class Config3:
    """Per-stage scheduling with `inflight` requests resident on the GPU
    (paper_2511_20975_b200.scheduler.SchedSession), mirrored by
    oracle/ref_bench.cpp run_sched for the reference arm."""

    def __init__(self, device: Device, inflight=10_000, rounds=200, seed=1, beam=4,
                 exhaustive=False):
        import torch

        self.dev, self.space = device, device.space
        self.inflight, self.rounds, self.seed, self.beam = inflight, rounds, seed, beam
        sp = self.space
        self.n, self.m = sp.n, sp.m
        reserve = inflight + rounds * 64 + 16
        batch = AccuracyBatch.generate(sp, GenParams(), reserve, seed)
        if exhaustive:
            res = device.route_enumerate_host(batch, OracleRouter())
            self.viable = [res.indices[res.offsets[r]:res.offsets[r + 1]] for r in range(reserve)]
        else:
            pred = ConfigPredictor(device)
            pr = pred.predict_batch(batch.to_device(device.torch_device), OracleRouter(0.002))
            torch.cuda.synchronize()
            nv = pr.n_viable.cpu().numpy()
            vv = pr.viable.cpu().numpy().view(np.uint32)
            self.viable = [vv[r, : nv[r]].copy() for r in range(reserve)]
        self.place = [self.m ** (self.n - 1 - a) for a in range(self.n)]
        self.sess = SchedSession(device, inflight + 64,
                                 sum(len(v) for v in self.viable) + 1)
        self.next_id = 0
        self.stages = {}   # slot -> stage list (host mirror)
        self._fill()

    def _make(self, rid):
        """Request rid with k = mix(12345, rid) % N stages already run."""
        v = np.asarray(self.viable[rid], np.uint32)
        st = [READY] + [PENDING] * (self.n - 1)
        k = mix(12345, rid) % self.n
        for a in range(k):
            digits = (v // self.place[a]) % self.m
            cands = np.unique(digits)
            mdl = int(cands[mix(12345, rid, a) % len(cands)])
            v = v[digits == mdl]
            st[a] = DONE
            st[a + 1] = READY
        return v, st

    def _fill(self):
        ids, arr, stages, viable = [], [], [], []
        while len(self.stages) + len(ids) < self.inflight:
            rid = self.next_id
            self.next_id += 1
            v, st = self._make(rid)
            ids.append(rid)
            arr.append(rid * 0.01)
            stages.extend(st)
            viable.append(v)
        if ids:
            slots = self.sess.add(Queue(self.n, ids, arr, stages, viable))
            for k, s in enumerate(slots):
                self.stages[int(s)] = stages[k * self.n:(k + 1) * self.n]

    def run(self, rounds=None, on_round=None):
        """Runs the loop; returns per-round decision latency (us) and the
        decision hash (same formula as ref_bench)."""
        weights = list(self.space.slot_throughput)
        self.dispatch_us = []
        h = GAMMA
        lat = []
        assigned = 0
        for rd in range(self.rounds if rounds is None else rounds):
            eng, _ = config3_engines(rd, self.seed, weights)
            t0 = time.perf_counter_ns()
            a = self.sess.round(eng, self.beam)
            t1 = time.perf_counter_ns()
            lat.append((t1 - t0) / 1e3)
            for (qi, rid, ag, mdl) in a.triples:
                h = mix(h, qi, rid, ag, mdl)
            assigned += len(a.triples)
            h = mix(h, int(a.utilization * 1e6) & MASK, a.states_explored, a.skips & MASK)
            if on_round:
                on_round(rd, a)
            # Request::mark_dispatched: the prefix prune that keeps the
            # candidate masks / histograms the next round reads current
            # (timed to the end of its kernel: the reference rebuilds this
            # RoundContext data inside beam_schedule, scheduler.cpp:294)
            t2 = time.perf_counter_ns()
            self.sess.dispatch(a)
            self.dev.synchronize()
            self.dispatch_us.append((time.perf_counter_ns() - t2) / 1e3)
            done = []
            for (qi, rid, ag, mdl), s in zip(a.triples, a.slots):
                self.sess.complete(s, ag)
                st = self.stages[s]
                st[ag] = DONE
                if ag + 1 < self.n:
                    st[ag + 1] = READY
                else:
                    done.append(s)
            if done:
                self.sess.remove(done)
                for s in done:
                    del self.stages[s]
                self._fill()
            # the dispatch / arrival kernels finish outside the next round's
            # timed decision
            self.dev.synchronize()
        return np.asarray(lat), h, assigned
