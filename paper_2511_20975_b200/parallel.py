"""Multi-GPU routing: request sharding and configuration-space sharding.

One process per GPU (torch.distributed, NCCL over NVLink).  The data path
has no collective: every rank enumerates its own shard.  The only exchange is
one all-gather of a fixed 32-byte record per (request, shard)

    {count (u64), best estimate (f64), best static cost (f64), best index (u64)}

from which every rank derives (a) the global CSR offsets of its members --
ranks own contiguous canonical-index ranges, so rank order is canonical order
and the concatenated lists equal the reference's sorted ViableSet
(predictor.cpp:256-259, accuracy.cpp:233-236) -- and (b) the per-input
runtime-cost choice, the minimum of (estimate, static cost, index)
(workload.cpp:149-176) over the shard minima.
"""
from __future__ import annotations

import numpy as np

REC_WORDS = 4  # u64 words per (request, shard) record


def shard_range(size: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) of canonical indices owned by `rank`."""
    base, rem = divmod(size, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def request_shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of requests owned by `rank` (request sharding)."""
    return shard_range(n, rank, world)


def pack_records(counts, best_est, best_cost, best_idx) -> np.ndarray:
    """[R, 4] uint64 records; doubles travel as their IEEE bit patterns."""
    R = len(counts)
    rec = np.zeros((R, REC_WORDS), np.uint64)
    rec[:, 0] = np.asarray(counts, np.uint64)
    rec[:, 1] = np.asarray(best_est, np.float64).view(np.uint64)
    rec[:, 2] = np.asarray(best_cost, np.float64).view(np.uint64)
    rec[:, 3] = np.asarray(best_idx, np.uint64)
    return rec


def merge_records(gathered: np.ndarray, rank: int):
    """gathered: [world, R, 4] records of every shard.  Returns (global
    counts [R], this rank's global offsets into each request's list [R], the
    winning (estimate, cost, index) per request)."""
    counts = gathered[:, :, 0].astype(np.uint64)
    total = counts.sum(axis=0)
    before = counts[:rank].sum(axis=0) if rank else np.zeros_like(total)
    est = gathered[:, :, 1].copy().view(np.float64)
    cost = gathered[:, :, 2].copy().view(np.float64)
    idx = gathered[:, :, 3]
    W, R = counts.shape
    best_e = np.full(R, np.inf)
    best_c = np.full(R, np.inf)
    best_i = np.full(R, np.iinfo(np.uint64).max, np.uint64)
    for w in range(W):  # lexicographic (estimate, cost, index) minimum
        has = counts[w] > 0
        e, c, i = est[w], cost[w], idx[w]
        better = has & ((e < best_e) | ((e == best_e) & ((c < best_c) | ((c == best_c) & (i < best_i)))))
        best_e = np.where(better, e, best_e)
        best_c = np.where(better, c, best_c)
        best_i = np.where(better, i, best_i)
    return total, before, (best_e, best_c, best_i)


def all_gather_records(rec: np.ndarray, group=None, device=None) -> np.ndarray:
    """One all-gather of host records (gloo on CPU ranks; the host mirror of
    exchange_records for tests and CPU-only callers)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return rec[None].copy()  # single process: nothing to exchange
    world = dist.get_world_size(group)
    t = torch.from_numpy(rec.view(np.int64).copy())
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return np.stack([p.cpu().numpy() for p in parts]).view(np.uint64)


def exchange_records(rec, world: int, group=None):
    """The one collective of the sharded path: all-gather of the [R, 4] int64
    record tensor into [world, R, 4] (NCCL over NVLink for device tensors,
    gloo for CPU tensors).  Enqueued on the caller's current stream, no host
    synchronisation."""
    import torch
    import torch.distributed as dist

    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return rec.unsqueeze(0)
    rec = rec.contiguous()
    out = torch.empty((world * rec.shape[0],) + tuple(rec.shape[1:]), dtype=rec.dtype, device=rec.device)
    dist.all_gather_into_tensor(out, rec, group=group)
    return out.view((world,) + tuple(rec.shape))


def shard_records(dev, res, n_requests: int, load_ctx=None, begin=None, end=None):
    """The [R, 4] int64 device records of this shard (ag_shard_records):
    {count, estimate bits, static-cost bits, index} of the runtime-cost
    minimum, or counts only without a load context.  When the routing result
    carries its verdict bitmap and the shard range is given, the records come
    straight from the bitmap (ag_select_bitmap: no member-list read)."""
    import ctypes as C

    import torch

    from ._capi import check, lib
    from .routing import _ptr
    from .scheduler import PER_INPUT_RUNTIME_COST

    rec = torch.zeros((max(n_requests, 1), REC_WORDS), dtype=torch.int64, device=dev.torch_device)
    if load_ctx is None:
        rec[:n_requests, 0] = res.counts[:n_requests].to(torch.int64)
        return rec[:n_requests]
    if res.bitmap is not None and begin is not None:
        from .scheduler import select_bitmap

        select_bitmap(dev, res.bitmap, res.counts[:n_requests], begin, end, PER_INPUT_RUNTIME_COST, load_ctx,
                      check_errors=False, records=rec)
        return rec[:n_requests]
    load = load_ctx.c()
    check(lib().ag_shard_records(dev.handle, C.c_void_p(_ptr(res.indices)), C.c_void_p(_ptr(res.offsets)),
                                 n_requests, PER_INPUT_RUNTIME_COST, C.byref(load), C.c_void_p(_ptr(rec))))
    return rec[:n_requests]


def merge_device(dev, gathered, rank: int):
    """ag_merge_records over the gathered [world, R, 4] records: (global
    counts, this rank's offsets, (best estimate, best static cost, best
    index)) as device tensors."""
    import ctypes as C

    import torch

    from ._capi import check, lib
    from .routing import _ptr

    world, R = int(gathered.shape[0]), int(gathered.shape[1])
    kw = dict(device=gathered.device)
    total = torch.empty(max(R, 1), dtype=torch.int64, **kw)
    before = torch.empty(max(R, 1), dtype=torch.int64, **kw)
    bi = torch.empty(max(R, 1), dtype=torch.int64, **kw)
    be = torch.empty(max(R, 1), dtype=torch.float64, **kw)
    bc = torch.empty(max(R, 1), dtype=torch.float64, **kw)
    check(lib().ag_merge_records(dev.handle, C.c_void_p(_ptr(gathered)), world, rank, R,
                                 *[C.c_void_p(_ptr(t)) for t in (total, before, bi, be, bc)]))
    return total[:R], before[:R], (be[:R], bc[:R], bi[:R])


def route_space_sharded(dev, truth_dev, router, rank, world, load_ctx=None, out=None, group=None):
    """Config 4: every rank enumerates its canonical-index shard of every
    request (ag_route_enumerate over [begin, end)), reduces it to one 32-byte
    record per request on the device (ag_select_bitmap from the verdict
    bitmap when `out` holds one, else ag_shard_records), then ONE all-gather
    of the records and a device-side merge (ag_merge_records).  No host
    round trip anywhere: everything is enqueued on the device's stream.
    Returns the local result, the global counts, this shard's global offsets
    and the global (estimate, static cost, index) choice, as device tensors
    (the choice is meaningful only with a load context)."""
    begin, end = shard_range(dev.space.size, rank, world)
    res = dev.route_enumerate(truth_dev, router, begin, end, out=out)
    R = truth_dev.n_requests
    rec = shard_records(dev, res, R, load_ctx, begin, end)
    gathered = exchange_records(rec, world, group)
    total, before, best = merge_device(dev, gathered, rank)
    return res, total, before, best
