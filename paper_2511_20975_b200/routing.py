"""Host-side mirror of the reference routing interface over the C ABI.

Reference API (paths relative to /root/reference/proj):
  * ConfigSpace / WorkflowGraph / ModelCatalog  include/aragog/workflow.h:34-152
  * AccurateSet / generate_accurate_set          include/aragog/accuracy.h:34-78
  * RouterBackend / OracleRouter / NoisyRouter   include/aragog/router.h:33-70
  * enumerate_members                            include/aragog/accuracy.h:81-82

Device buffers are torch CUDA tensors (plumbing only); every computation runs
in the CUDA kernels of libaragog_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import check, lib

INF = float("inf")


def _ptr(a) -> int | None:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data if a.size else None
    return a.data_ptr() if a.numel() else None


class ConfigSpace:
    """WorkflowGraph::build + ModelCatalog + ConfigSpace (workflow.cpp:38-224)."""

    def __init__(self, n_agents: int, edges, cost, slot_throughput):
        e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2) if len(edges) else
                                 np.zeros((0, 2), np.int32))
        cost = np.ascontiguousarray(cost, np.float64)
        w = np.ascontiguousarray(slot_throughput, np.float64)
        h = C.c_void_p()
        check(lib().ag_space_create(n_agents, len(e), C.c_void_p(_ptr(e)), len(cost),
                                    C.c_void_p(_ptr(cost)), C.c_void_p(_ptr(w)), C.byref(h)))
        self._h = h
        self.cost = cost
        self.slot_throughput = w
        n, m, size = C.c_int32(), C.c_int32(), C.c_uint64()
        decl = np.zeros(n_agents, np.int32)
        depth = np.zeros(n_agents, np.int32)
        check(lib().ag_space_info(h, C.byref(n), C.byref(m), C.c_void_p(_ptr(decl)),
                                  C.c_void_p(_ptr(depth)), C.byref(size)))
        self.n, self.m, self.size = n.value, m.value, size.value
        self.decl, self.depth = decl, depth

    @classmethod
    def chain(cls, n: int, m: int, cost=None, slot_throughput=None):
        """An n-agent chain a0 -> ... -> a{n-1} over m tiers.  Default catalog:
        cost x1.5 and weight /1.5 per tier."""
        if cost is None:
            cost = [1.5 ** i for i in range(m)]
        if slot_throughput is None:
            slot_throughput = [8.0 / 1.5 ** i for i in range(m)]
        return cls(n, [(i - 1, i) for i in range(1, n)], cost, slot_throughput)

    @property
    def handle(self):
        return self._h

    def index_of(self, digits) -> int:
        idx = 0
        for d in digits:
            idx = idx * self.m + int(d)
        return idx

    def at_index(self, idx: int) -> list[int]:
        out = [0] * self.n
        for i in range(self.n - 1, -1, -1):
            out[i] = idx % self.m
            idx //= self.m
        return out

    @property
    def top(self) -> int:
        return self.size - 1

    def __del__(self):
        try:  # module globals may already be gone at interpreter shutdown
            _capi.release("ag_space_destroy", getattr(self, "_h", None))
        except Exception:  # noqa: BLE001
            pass
        self._h = None


@dataclass
class GenParams:
    """AccuracyGenParams (include/aragog/accuracy.h:42-52)."""
    p_easy: float = 0.6
    p_medium: float = 0.3
    p_hard: float = 0.1
    easy_base_prob: float = 0.5
    violation_rate: float = 0.0


class AccuracyBatch:
    """A batch of AccurateSets in CSR form (host numpy arrays)."""

    def __init__(self, n, request_ids, seed_ptr, seeds, removed_ptr, removed):
        self.n = n
        self.request_ids = np.ascontiguousarray(request_ids, np.uint64)
        self.seed_ptr = np.ascontiguousarray(seed_ptr, np.int32)
        self.seeds = np.ascontiguousarray(np.asarray(seeds, np.uint8).reshape(-1))
        self.removed_ptr = np.ascontiguousarray(removed_ptr, np.int32)
        self.removed = np.ascontiguousarray(np.asarray(removed, np.uint64).reshape(-1))

    @property
    def n_requests(self) -> int:
        return len(self.request_ids)

    @classmethod
    def from_lists(cls, n, seeds_list, removed_list, request_ids=None):
        R = len(seeds_list)
        sp = np.zeros(R + 1, np.int32)
        rp = np.zeros(R + 1, np.int32)
        for i, s in enumerate(seeds_list):
            sp[i + 1] = sp[i] + len(s)
        for i, r in enumerate(removed_list):
            rp[i + 1] = rp[i] + len(r)
        seeds = (np.concatenate([np.asarray(s, np.uint8).reshape(-1, n) for s in seeds_list if len(s)])
                 if sp[-1] else np.zeros((0, n), np.uint8))
        rem = (np.concatenate([np.asarray(r, np.uint64).reshape(-1) for r in removed_list if len(r)])
               if rp[-1] else np.zeros(0, np.uint64))
        ids = np.arange(R, dtype=np.uint64) if request_ids is None else request_ids
        return cls(n, ids, sp, seeds, rp, rem)

    @classmethod
    def generate(cls, space: ConfigSpace, params: GenParams, count: int, seed: int,
                 salt: int = 0xA2, first_id: int = 0):
        """generate_accuracy_table rows first_id.. (accuracy.cpp:144-225)."""
        gp = _capi.GenParams(params.p_easy, params.p_medium, params.p_hard,
                             params.easy_base_prob, params.violation_rate)
        sp = np.zeros(count + 1, np.int32)
        rp = np.zeros(count + 1, np.int32)
        seeds_cap = 2 * count + 1
        seeds = np.zeros((seeds_cap, space.n), np.uint8)
        rem_cap = count * min(space.size, 4096) + 1 if params.violation_rate > 0 else 1
        removed = np.zeros(rem_cap, np.uint64)
        check(lib().ag_generate_truth(space.handle, C.byref(gp), C.c_uint64(seed), C.c_uint64(salt),
                                      C.c_uint64(first_id), count, C.c_void_p(_ptr(sp)),
                                      C.c_void_p(_ptr(seeds)), seeds_cap, C.c_void_p(_ptr(rp)),
                                      C.c_void_p(_ptr(removed)), rem_cap))
        ids = np.arange(first_id, first_id + count, dtype=np.uint64)
        return cls(space.n, ids, sp, seeds[: sp[-1]], rp, removed[: rp[-1]])

    def seeds_of(self, r):
        return self.seeds[self.seed_ptr[r] * self.n: self.seed_ptr[r + 1] * self.n].reshape(-1, self.n)

    def removed_of(self, r):
        return self.removed[self.removed_ptr[r]: self.removed_ptr[r + 1]]

    def slice(self, lo, hi) -> "AccuracyBatch":
        s0, s1 = self.seed_ptr[lo], self.seed_ptr[hi]
        r0, r1 = self.removed_ptr[lo], self.removed_ptr[hi]
        return AccuracyBatch(self.n, self.request_ids[lo:hi], self.seed_ptr[lo:hi + 1] - s0,
                             self.seeds[s0 * self.n: s1 * self.n], self.removed_ptr[lo:hi + 1] - r0,
                             self.removed[r0:r1])

    def c_struct(self) -> _capi.Truth:
        return _capi.Truth(self.n_requests, _ptr(self.request_ids), _ptr(self.seed_ptr),
                           _ptr(self.seeds), _ptr(self.removed_ptr), _ptr(self.removed))

    def to_device(self, device="cuda") -> "DeviceAccuracyBatch":
        return DeviceAccuracyBatch(self, device)


class DeviceAccuracyBatch:
    """The same CSR resident in HBM (torch tensors as allocations)."""

    def __init__(self, host: AccuracyBatch, device="cuda"):
        import torch

        self.n = host.n

        def put(a, dt):
            t = torch.from_numpy(np.ascontiguousarray(a).view(dt) if a.size else np.zeros(1, dt))
            return t.to(device)

        self.request_ids = put(host.request_ids, np.int64)
        self.seed_ptr = put(host.seed_ptr, np.int32)
        self.seeds = put(host.seeds, np.uint8)
        self.removed_ptr = put(host.removed_ptr, np.int32)
        self.removed = put(host.removed, np.int64)
        self.n_requests = host.n_requests

    def c_struct(self) -> _capi.Truth:
        return _capi.Truth(self.n_requests, _ptr(self.request_ids), _ptr(self.seed_ptr),
                           _ptr(self.seeds), _ptr(self.removed_ptr), _ptr(self.removed))


def OracleRouter(eval_latency: float = 0.0) -> _capi.Router:
    """OracleRouter (router.h:43-53)."""
    return _capi.Router(_capi.AG_ROUTER_ORACLE, 0.0, 0.0, 0, eval_latency)


def NoisyRouter(false_positive_rate: float, false_negative_rate: float, seed: int,
                eval_latency: float = 0.0) -> _capi.Router:
    """NoisyRouter over the oracle (router.h:57-70)."""
    return _capi.Router(_capi.AG_ROUTER_NOISY, false_positive_rate, false_negative_rate, seed,
                        eval_latency)


@dataclass
class RouteResult:
    counts: object        # [R] uint64 (int64 tensor / numpy)
    offsets: object       # [R+1]
    indices: object       # members, canonical order, CSR by offsets (or None)
    bitmap: object        # [R, W] uint32 words (or None)

    def members(self, r):
        o = self.offsets
        lo, hi = int(o[r]), int(o[r + 1])
        return self.indices[lo:hi]


class Device:
    """An ag_ctx bound to one space and one CUDA device."""

    def __init__(self, space: ConfigSpace, device: int = 0, stream=None):
        import torch

        self.space = space
        self.device = device
        h = C.c_void_p()
        check(lib().ag_ctx_create(space.handle, device, C.byref(h)))
        self._h = h
        self.torch_device = torch.device("cuda", device)
        self.set_stream(stream if stream is not None else torch.cuda.current_stream(device))

    def set_stream(self, stream):
        self.stream = stream
        check(lib().ag_ctx_set_stream(self._h, C.c_void_p(stream.cuda_stream)))

    @property
    def handle(self):
        return self._h

    @property
    def launch_count(self) -> int:
        return int(lib().ag_ctx_launch_count(self._h))

    def synchronize(self):
        check(lib().ag_ctx_synchronize(self._h))

    def profile_begin(self):
        """Start the live per-kernel CUDA-event profile (ag_ctx_profile_begin)."""
        check(lib().ag_ctx_profile_begin(self._h))

    def profile_end(self) -> dict:
        """{kernel name: (total device ms, launches)} since profile_begin."""
        k = 11  # AG_NUM_KERNELS
        ms = (C.c_double * k)()
        n = (C.c_uint64 * k)()
        check(lib().ag_ctx_profile_end(self._h, ms, n))
        name = lib().ag_kernel_name
        name.restype = C.c_char_p
        return {name(i).decode(): (ms[i], int(n[i])) for i in range(k) if n[i]}

    # ------------------------------------------------------------ routing
    def alloc_route(self, n_requests, begin, end, capacity, bitmap=False):
        import torch

        W = (end - begin + 31) // 32
        dev = self.torch_device
        return dict(
            counts=torch.zeros(n_requests, dtype=torch.int64, device=dev),
            offsets=torch.zeros(n_requests + 1, dtype=torch.int64, device=dev),
            indices=(torch.zeros(max(capacity, 1), dtype=torch.int32, device=dev)
                     if capacity is not None else None),
            bitmap=(torch.zeros((n_requests, max(W, 1)), dtype=torch.int32, device=dev)
                    if bitmap else None),
            overflow=torch.zeros(1, dtype=torch.int32, device=dev),
            capacity=0 if capacity is None else capacity)

    def route_enumerate(self, truth: DeviceAccuracyBatch, router, begin=0, end=None,
                        force_top=False, out=None, capacity=None, bitmap=False,
                        compact=True) -> RouteResult:
        """Enumerate mode on device buffers (async on the context stream)."""
        end = self.space.size if end is None else end
        if out is None:
            if compact and capacity is None:
                capacity = truth.n_requests * (end - begin)
            out = self.alloc_route(truth.n_requests, begin, end, capacity if compact else None,
                                   bitmap)
        t = truth.c_struct()
        ro = _capi.RouteOut(_ptr(out["bitmap"]), _ptr(out["counts"]), _ptr(out["offsets"]),
                            _ptr(out["indices"]), out["capacity"], _ptr(out["overflow"]))
        check(lib().ag_route_enumerate(self._h, C.byref(t), C.byref(router), C.c_uint64(begin),
                                       C.c_uint64(end), C.c_uint32(_capi.AG_FORCE_TOP if force_top else 0),
                                       C.byref(ro)))
        self._last_out = out
        return RouteResult(out["counts"], out["offsets"], out["indices"], out["bitmap"])

    def route_linear(self, emb, heads, bias, begin=0, end=None, force_top=False, out=None,
                     capacity=None, bitmap=False) -> RouteResult:
        """Enumerate mode with the learned router (ag_route_linear): device
        tensors emb [R, D] bf16, heads [space size, D] bf16, bias [size] f32;
        verdict = emb . heads[c] + bias[c] > 0 (async on the context stream)."""
        import torch

        end = self.space.size if end is None else end
        R = int(emb.shape[0])
        if out is None:
            out = self.alloc_route(R, begin, end, R * (end - begin) if capacity is None else capacity,
                                   bitmap)
        assert emb.dtype == torch.bfloat16 and heads.dtype == torch.bfloat16
        assert bias.dtype == torch.float32
        lh = _capi.LinearHeads(int(heads.shape[1]), _ptr(heads), _ptr(bias))
        ro = _capi.RouteOut(_ptr(out["bitmap"]), _ptr(out["counts"]), _ptr(out["offsets"]),
                            _ptr(out["indices"]), out["capacity"], _ptr(out["overflow"]))
        check(lib().ag_route_linear(self._h, C.c_void_p(_ptr(emb)), R, C.byref(lh), C.c_uint64(begin),
                                    C.c_uint64(end),
                                    C.c_uint32(_capi.AG_FORCE_TOP if force_top else 0), C.byref(ro)))
        self._last_out = (out, emb, heads, bias)
        return RouteResult(out["counts"], out["offsets"], out["indices"], out["bitmap"])

    def route_enumerate_host(self, truth: AccuracyBatch, router, begin=0, end=None,
                             force_top=False, capacity=None, indices=None, counts=None,
                             offsets=None):
        """Enumerate mode with host buffers, copies included (the e2e path)."""
        end = self.space.size if end is None else end
        R = truth.n_requests
        counts = np.zeros(R, np.uint64) if counts is None else counts
        offsets = np.zeros(R + 1, np.uint64) if offsets is None else offsets
        if indices is None:
            cap = R * (end - begin) if capacity is None else capacity
            indices = np.zeros(max(cap, 1), np.uint32)
        total = C.c_uint64()
        t = truth.c_struct()
        check(lib().ag_route_enumerate_host(
            self._h, C.byref(t), C.byref(router), C.c_uint64(begin), C.c_uint64(end),
            C.c_uint32(_capi.AG_FORCE_TOP if force_top else 0), C.c_void_p(_ptr(counts)),
            C.c_void_p(_ptr(offsets)), C.c_void_p(_ptr(indices)), C.c_uint64(len(indices)),
            C.byref(total)))
        return RouteResult(counts, offsets, indices[: total.value], None)

    def __del__(self):
        try:  # module globals may already be gone at interpreter shutdown
            _capi.release("ag_ctx_destroy", getattr(self, "_h", None))
        except Exception:  # noqa: BLE001
            pass
        self._h = None


def enumerate_members(space: ConfigSpace, seeds, removed=(), device: Device | None = None):
    """enumerate_members (accuracy.cpp:227-238): members of one AccurateSet in
    canonical order, computed on the GPU.  Keeps the reference's 4096-config
    guard (accuracy.cpp:229-231); use Device.route_enumerate for larger spaces."""
    if space.size == 0 or space.size > 4096:
        raise _capi.ValidationError(_capi.AG_ERR_VALIDATION,
                                    "configuration space too large to enumerate")
    dev = device or Device(space)
    batch = AccuracyBatch.from_lists(space.n, [seeds], [list(removed)])
    res = dev.route_enumerate_host(batch, OracleRouter())
    return [space.at_index(int(i)) for i in res.indices]
