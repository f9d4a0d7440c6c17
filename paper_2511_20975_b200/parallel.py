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
    """One all-gather of the per-shard records (NCCL on GPUs, gloo on CPU)."""
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


def route_space_sharded(dev, truth_dev, router, rank, world, load_ctx=None, out=None):
    """Config 4: every rank enumerates its canonical-index shard of every
    request, then one all-gather of per-shard records.  Returns the local
    result, the global counts, this shard's global offsets, and (with a load
    context) the global runtime-cost choice."""
    import torch

    from .scheduler import PER_INPUT_RUNTIME_COST, select_per_input

    begin, end = shard_range(dev.space.size, rank, world)
    res = dev.route_enumerate(truth_dev, router, begin, end, out=out)
    R = truth_dev.n_requests
    counts = res.counts.cpu().numpy().astype(np.uint64)
    if load_ctx is not None:
        nz = counts > 0
        ch, est = select_per_input(dev, res.indices, res.offsets, PER_INPUT_RUNTIME_COST, load_ctx) \
            if nz.all() else _select_nonempty(dev, res, load_ctx, nz)
        best_i = ch.cpu().numpy().view(np.uint32).astype(np.uint64)
        best_e = est.cpu().numpy()
        cost = np.asarray(dev.space.cost)
        digits = [(best_i // dev.space.m ** (dev.space.n - 1 - a)) % dev.space.m
                  for a in range(dev.space.n)]
        best_c = np.zeros(R)
        for d in digits:  # static_cost: left fold in agent order
            best_c = best_c + cost[d.astype(np.int64)]
    else:
        best_e = np.zeros(R)
        best_c = np.zeros(R)
        best_i = np.zeros(R, np.uint64)
    rec = pack_records(counts, best_e, best_c, best_i)
    torch.cuda.synchronize()
    gathered = all_gather_records(rec, device=dev.torch_device)
    total, before, best = merge_records(gathered, rank)
    return res, total, before, best


def _select_nonempty(dev, res, load_ctx, nz):
    """select_per_input over the requests whose shard is non-empty."""
    import torch

    from .scheduler import PER_INPUT_RUNTIME_COST, select_per_input

    R = len(nz)
    ch = torch.zeros(R, dtype=torch.int32, device=dev.torch_device)
    est = torch.full((R,), float("inf"), dtype=torch.float64, device=dev.torch_device)
    ids = np.nonzero(nz)[0]
    if len(ids):
        offs = res.offsets.cpu().numpy()
        sub_offs = np.concatenate([[0], np.cumsum(offs[ids + 1] - offs[ids])]).astype(np.int64)
        parts = [res.indices[int(offs[r]):int(offs[r + 1])] for r in ids]
        mem = torch.cat(parts)
        c2, e2 = select_per_input(dev, mem, torch.from_numpy(sub_offs).to(dev.torch_device),
                                  PER_INPUT_RUNTIME_COST, load_ctx)
        ch[torch.from_numpy(ids).to(dev.torch_device)] = c2
        est[torch.from_numpy(ids).to(dev.torch_device)] = e2
    return ch, est
