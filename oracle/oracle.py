"""TEST INFRASTRUCTURE ONLY: ctypes binding for the plain-C oracle restatement.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module; the product package (paper_2511_20975_b200) never does.  Each
wrapper names the reference function it restates (see aragog_oracle.c).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")

ORACLE, NOISY = 0, 1
PENDING, READY, INFLIGHT, DONE = 0, 1, 2, 3


def build():
    subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])


def _lib():
    global _L
    try:
        return _L
    except NameError:
        pass
    if not os.path.exists(LIB_PATH):
        build()
    _L = C.CDLL(LIB_PATH)
    _L.ago_last_error.restype = C.c_char_p
    _L.ago_mix.restype = C.c_uint64
    _L.ago_enumerate.restype = C.c_uint64
    _L.ago_prefix_prune.restype = C.c_int64
    return _L


class GenParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("p_easy", "p_medium", "p_hard", "easy_base_prob", "violation_rate")]


class Router(C.Structure):
    _fields_ = [("kind", C.c_int), ("fp", C.c_double), ("fn", C.c_double),
                ("noise_seed", C.c_uint64), ("eval_latency", C.c_double)]


class Truth(C.Structure):
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("n_requests", C.c_int),
                ("request_ids", C.c_void_p), ("seed_ptr", C.c_void_p), ("seeds", C.c_void_p),
                ("removed_ptr", C.c_void_p), ("removed", C.c_void_p)]


class Prediction(C.Structure):
    _fields_ = [("search_evals", C.c_int), ("verify_evals", C.c_int), ("truncated", C.c_int),
                ("router_time", C.c_double), ("n_viable", C.c_int)]


class Load(C.Structure):
    _fields_ = [("n_tiers", C.c_int), ("occupancy", C.c_void_p), ("queued_ahead", C.c_void_p),
                ("slots", C.c_void_p), ("mean", C.c_void_p)]


class Queue(C.Structure):
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("depth", C.c_void_p), ("decl", C.c_void_p),
                ("n_requests", C.c_int), ("ids", C.c_void_p), ("arrival", C.c_void_p),
                ("stages", C.c_void_p), ("viable_ptr", C.c_void_p), ("viable", C.c_void_p)]


class Engines(C.Structure):
    _fields_ = [("n_engines", C.c_int), ("model", C.c_void_p), ("slots", C.c_void_p),
                ("occupancy", C.c_void_p), ("weight", C.c_void_p)]


class Triple(C.Structure):
    _fields_ = [("request_index", C.c_int32), ("agent", C.c_int32), ("model", C.c_int32),
                ("pad", C.c_int32), ("request_id", C.c_uint64)]


class Assignment(C.Structure):
    _fields_ = [("n_triples", C.c_int), ("utilization", C.c_double), ("flexibility", C.c_double),
                ("skips", C.c_int64), ("states_explored", C.c_uint64)]


class Snapshot(C.Structure):
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("n_requests", C.c_int), ("n_engines", C.c_int),
                ("depth", C.c_int32 * 8), ("decl", C.c_int32 * 8),
                ("cost", C.c_double * 4), ("weight", C.c_double * 4),
                ("eng_model", C.c_int32 * 4), ("eng_slots", C.c_int32 * 4), ("eng_occ", C.c_int32 * 4),
                ("eng_weight", C.c_double * 4), ("ids", C.c_uint64 * 8), ("arrival", C.c_double * 8),
                ("stages", C.c_uint8 * 64), ("viable_ptr", C.c_int64 * 9), ("viable", C.c_uint64 * 2048)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, _lib().ago_last_error().decode())


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


def mix(words):
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return int(_lib().ago_mix(C.c_void_p(_p(w)), len(w)))


def graph_build(n, edges):
    """WorkflowGraph::build -> (decl order per canonical pos, depth, pred masks, succ masks)."""
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1))
    order = np.zeros(n, np.int32)
    depth = np.zeros(n, np.int32)
    pred = np.zeros(max(n, 1), np.uint64)
    succ = np.zeros(max(n, 1), np.uint64)
    _check(_lib().ago_graph_build(n, len(e) // 2, C.c_void_p(_p(e)), C.c_void_p(_p(order)),
                                  C.c_void_p(_p(depth)), C.c_void_p(_p(pred)), C.c_void_p(_p(succ))))
    return order, depth, pred, succ


def gen_truth(n, m, params, seed, request_id, salt=0xA2):
    """generate_accurate_set -> (tier, seeds[k,n] uint8, removed uint64)."""
    gp = GenParams(*params)
    seeds = np.zeros((16, n), np.uint8)
    removed = np.zeros(4096, np.uint64)
    ns, nr, tier = C.c_int(), C.c_int(), C.c_int()
    _check(_lib().ago_gen_truth(n, m, C.byref(gp), C.c_uint64(seed), C.c_uint64(request_id),
                                C.c_uint64(salt), C.c_void_p(_p(seeds)), 16, C.byref(ns),
                                C.c_void_p(_p(removed)), 4096, C.byref(nr), C.byref(tier)))
    return tier.value, seeds[: ns.value].copy(), removed[: nr.value].copy()


class TruthBatch:
    """A batch of AccurateSets in the CSR layout shared with the CUDA ABI."""

    def __init__(self, n, m, seeds_list, removed_list, request_ids=None):
        self.n, self.m = n, m
        R = len(seeds_list)
        self.request_ids = np.ascontiguousarray(
            np.arange(R, dtype=np.uint64) if request_ids is None else np.asarray(request_ids, np.uint64))
        self.seed_ptr = np.zeros(R + 1, np.int32)
        self.removed_ptr = np.zeros(R + 1, np.int32)
        for i, s in enumerate(seeds_list):
            self.seed_ptr[i + 1] = self.seed_ptr[i] + len(s)
        for i, r in enumerate(removed_list):
            self.removed_ptr[i + 1] = self.removed_ptr[i] + len(r)
        self.seeds = np.ascontiguousarray(
            np.concatenate([np.asarray(s, np.uint8).reshape(-1, n) for s in seeds_list]) if R else
            np.zeros((0, n), np.uint8)).reshape(-1)
        rem = [np.asarray(r, np.uint64).reshape(-1) for r in removed_list]
        self.removed = np.ascontiguousarray(np.concatenate(rem) if rem else np.zeros(0, np.uint64))
        if self.removed.size == 0:
            self.removed = np.zeros(1, np.uint64)
        if self.seeds.size == 0:
            self.seeds = np.zeros(1, np.uint8)
        self.n_requests = R

    def c(self):
        return Truth(self.n, self.m, self.n_requests, _p(self.request_ids), _p(self.seed_ptr),
                     _p(self.seeds), _p(self.removed_ptr), _p(self.removed))


def router_eval(tb, router, req, index):
    t = tb.c()
    return int(_lib().ago_router_eval(C.byref(t), C.byref(router), req, C.c_uint64(index)))


def enumerate_bitmap(tb, router, req, begin, end, force_top=False):
    """Enumerate-mode verdict bitmap over [begin, end) -> (count, uint32 words)."""
    t = tb.c()
    words = np.zeros((end - begin + 31) // 32, np.uint32)
    cnt = _lib().ago_enumerate(C.byref(t), C.byref(router), req, C.c_uint64(begin), C.c_uint64(end),
                               int(force_top), C.c_void_p(_p(words)))
    return int(cnt), words


def build_chains(n, m, chain_cap=0, exhaustive_limit=4096, cap=1 << 16):
    L = n * (m - 1) + 1
    out = np.zeros(cap * L, np.uint64)
    ex = C.c_int()
    k = _lib().ago_build_chains(n, m, chain_cap, C.c_uint64(exhaustive_limit), C.c_void_p(_p(out)),
                                cap, C.byref(ex))
    if k < 0:
        raise OracleError(2, "chain cap too small")
    return out[: k * L].reshape(k, L).copy(), bool(ex.value)


def predict(tb, router, cost, chains, req, budget):
    t = tb.c()
    cost = np.ascontiguousarray(cost, np.float64)
    ch = np.ascontiguousarray(chains, np.uint64)
    cap = ch.size + 2
    out = np.zeros(cap, np.uint64)
    res = Prediction()
    _check(_lib().ago_predict(C.byref(t), C.byref(router), C.c_void_p(_p(cost)), C.c_void_p(_p(ch)),
                              ch.shape[0], req, C.c_double(budget), C.c_void_p(_p(out)), cap,
                              C.byref(res)))
    return dict(viable=out[: res.n_viable].copy(), search_evals=res.search_evals,
                verify_evals=res.verify_evals, router_time=res.router_time,
                truncated=bool(res.truncated))


def estimate_completion(occupancy, queued, slots, mean, digits):
    arrs = [np.ascontiguousarray(a, t) for a, t in ((occupancy, np.int32), (queued, np.int32),
                                                     (slots, np.int32), (mean, np.float64))]
    ld = Load(len(arrs[2]), *[_p(a) for a in arrs])
    d = np.ascontiguousarray(digits, np.uint8)
    out = C.c_double()
    _check(_lib().ago_estimate_completion(C.byref(ld), len(d), C.c_void_p(_p(d)), C.byref(out)))
    return out.value


def select_per_input(n, m, cost, occupancy, queued, slots, mean, kind, members):
    arrs = [np.ascontiguousarray(a, t) for a, t in ((occupancy, np.int32), (queued, np.int32),
                                                     (slots, np.int32), (mean, np.float64))]
    ld = Load(len(arrs[2]), *[_p(a) for a in arrs])
    cost = np.ascontiguousarray(cost, np.float64)
    mem = np.ascontiguousarray(members, np.uint64)
    chosen, est = C.c_uint64(), C.c_double()
    _check(_lib().ago_select_per_input(n, m, C.c_void_p(_p(cost)), C.byref(ld), kind,
                                       C.c_void_p(_p(mem)), len(mem), C.byref(chosen), C.byref(est)))
    return int(chosen.value), est.value


def select_per_workflow(n, m, cost, tb, tolerance=0.0):
    """select_per_workflow_config (reference src/workload.cpp:99-127), restated:
    every configuration in (static cost, canonical index) order -- the cost a
    left fold in agent order (workflow.cpp:291-296) -- and the first one
    accurate on at least (1 - tolerance) * |sample| sets.  The membership
    verdicts come from the C restatement's enumerate (AccurateSet::contains).
    Test infrastructure only."""
    R = len(tb.request_ids)
    if R == 0:
        raise ValueError("per-workflow sample is empty")
    S = m ** n
    hits = np.zeros(S, np.int64)
    for r in range(R):
        cnt, words = enumerate_bitmap(tb, Router(ORACLE, 0, 0, 0, 0), r, 0, S)
        bits = np.unpackbits(np.asarray(words, np.uint32).view(np.uint8), bitorder="little")[:S]
        hits += bits
    costs = np.zeros(S)
    idx = np.arange(S, dtype=np.int64)
    for a in range(n):  # agent order, left fold
        digit = (idx // (m ** (n - 1 - a))) % m
        costs = costs + np.asarray(cost, np.float64)[digit]
    needed = (1.0 - tolerance) * float(R)
    order = np.lexsort((idx, costs))
    for c in order:
        if float(hits[c]) >= needed:
            return int(c), int(hits[c])
    raise ValueError("per-workflow scan found no configuration")


class QueueData:
    """Flat queue view (the reference's vector<const Request*>) + engine pools."""

    def __init__(self, n, m, depth, decl, ids, arrival, stages, viable_lists,
                 eng_model, eng_slots, eng_occ, eng_weight):
        self.n, self.m = n, m
        self.depth = np.ascontiguousarray(depth, np.int32)
        self.decl = np.ascontiguousarray(decl, np.int32)
        self.ids = np.ascontiguousarray(ids, np.uint64)
        self.arrival = np.ascontiguousarray(arrival, np.float64)
        self.stages = np.ascontiguousarray(np.asarray(stages, np.uint8).reshape(-1))
        ptr = [0]
        for v in viable_lists:
            ptr.append(ptr[-1] + len(v))
        self.viable_ptr = np.asarray(ptr, np.int64)
        self.viable = np.ascontiguousarray(
            np.concatenate([np.asarray(v, np.uint64) for v in viable_lists]) if viable_lists else
            np.zeros(1, np.uint64))
        if self.viable.size == 0:
            self.viable = np.zeros(1, np.uint64)
        self.eng_model = np.ascontiguousarray(eng_model, np.int32)
        self.eng_slots = np.ascontiguousarray(eng_slots, np.int32)
        self.eng_occ = np.ascontiguousarray(eng_occ, np.int32)
        self.eng_weight = np.ascontiguousarray(eng_weight, np.float64)

    @property
    def n_requests(self):
        return len(self.ids)

    def cq(self):
        return Queue(self.n, self.m, _p(self.depth), _p(self.decl), len(self.ids), _p(self.ids),
                     _p(self.arrival), _p(self.stages), _p(self.viable_ptr), _p(self.viable))

    def ce(self):
        return Engines(len(self.eng_model), _p(self.eng_model), _p(self.eng_slots),
                       _p(self.eng_occ), _p(self.eng_weight))


def two_level_order(qd):
    q = qd.cq()
    cap = max(1, int((qd.stages == READY).sum()))
    pr = np.zeros(cap, np.int32)
    pa = np.zeros(cap, np.int32)
    npairs = C.c_int()
    _check(_lib().ago_two_level_order(C.byref(q), C.c_void_p(_p(pr)), C.c_void_p(_p(pa)), cap,
                                      C.byref(npairs)))
    return pr[: npairs.value].copy(), pa[: npairs.value].copy()


def beam_schedule(qd, width):
    q, e = qd.cq(), qd.ce()
    cap = max(1, int((qd.stages == READY).sum()))
    tr = (Triple * cap)()
    occ = np.zeros(max(1, len(qd.eng_model)), np.int32)
    out = Assignment()
    _check(_lib().ago_beam_schedule(C.byref(q), C.byref(e), width, tr, cap, C.c_void_p(_p(occ)),
                                    C.byref(out)))
    triples = [(tr[i].request_index, tr[i].request_id, tr[i].agent, tr[i].model)
               for i in range(out.n_triples)]
    return dict(triples=triples, occupancy=occ[: len(qd.eng_model)].tolist(),
                utilization=out.utilization, flexibility=out.flexibility, skips=out.skips,
                states_explored=out.states_explored)


def audit_round_fairness(qd, triples):
    """audit_round_fairness (scheduler.cpp:456-480): triples as
    (request_index, request_id, agent, model); returns [(RequestId, agent)]."""
    q, e = qd.cq(), qd.ce()
    n = len(triples)
    tr = (Triple * max(1, n))()
    for i, (qi, rid, a, mdl) in enumerate(triples):
        tr[i].request_index, tr[i].request_id, tr[i].agent, tr[i].model = qi, rid, a, mdl
    cap = max(1, int((qd.stages == READY).sum()))
    ids = np.zeros(cap, np.uint64)
    ags = np.zeros(cap, np.int32)
    nv = C.c_int()
    _check(_lib().ago_audit_round_fairness(C.byref(q), C.byref(e), tr, n, C.c_void_p(_p(ids)),
                                           C.c_void_p(_p(ags)), cap, C.byref(nv)))
    return [(int(ids[i]), int(ags[i])) for i in range(min(nv.value, cap))]


def generate_snapshot(seed, index):
    s = Snapshot()
    _check(_lib().ago_generate_snapshot(C.c_uint64(seed), C.c_uint64(index), C.byref(s)))
    n, R = s.n, s.n_requests
    vp = list(s.viable_ptr)[: R + 1]
    viable = [list(s.viable)[vp[i]: vp[i + 1]] for i in range(R)]
    return dict(n=n, m=s.m, depth=list(s.depth)[:n], decl=list(s.decl)[:n],
                ids=list(s.ids)[:R], arrival=list(s.arrival)[:R],
                stages=list(s.stages)[: R * n], viable=viable,
                eng_model=list(s.eng_model)[: s.n_engines], eng_slots=list(s.eng_slots)[: s.n_engines],
                eng_occ=list(s.eng_occ)[: s.n_engines], eng_weight=list(s.eng_weight)[: s.n_engines])


def prefix_prune(n, m, viable, agent, model):
    v = np.ascontiguousarray(viable, np.uint64).copy()
    k = _lib().ago_prefix_prune(n, m, C.c_void_p(_p(v)), len(v), agent, model)
    return None if k < 0 else v[:k]


def linear_logits(emb, heads, bias):
    """The learned router of SURVEY.md §8(f) rank 3 (not in the reference):
    logit(r, c) = emb[r] . heads[c] + bias[c], verdict = logit > 0, in fp64
    from the bf16 inputs (given as float arrays).  Test infrastructure only."""
    return np.asarray(emb, np.float64) @ np.asarray(heads, np.float64).T + np.asarray(bias, np.float64)[None, :]
