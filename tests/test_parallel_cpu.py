"""Multi-rank logic of the sharded routing path on CPU (gloo, world size 2):
shard ranges, the per-shard record all-gather, global offsets and the global
runtime-cost choice, checked against the C oracle over the whole space."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_20975_b200 import parallel as PL


def test_shard_ranges_partition():
    for size in (1, 7, 27, 32768, 12 ** 8):
        for world in (1, 2, 3, 4, 8):
            ranges = [PL.shard_range(size, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == size
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and a <= b


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_20975_b200 as P
        from oracle import oracle as O
        n, m, R = 4, 5, 12
        space = P.ConfigSpace.chain(n, m)
        batch = P.AccuracyBatch.generate(space, P.GenParams(), R, seed=4)
        tb = O.TruthBatch(n, m, [batch.seeds_of(r) for r in range(R)],
                          [batch.removed_of(r) for r in range(R)], batch.request_ids)
        b, e = PL.shard_range(space.size, rank, world)
        occ, queued, slots = [1, 0, 2, 0, 1], [3, 0, 1, 2, 0], [2, 2, 3, 1, 4]
        mean = [0.5 + 0.25 * i for i in range(m)]
        counts, best_e, best_c, best_i = [], [], [], []
        for r in range(R):
            cnt, words = O.enumerate_bitmap(tb, O.Router(0, 0, 0, 0, 0), r, b, e)
            bits = np.unpackbits(words.view(np.uint8), bitorder="little")
            members = (np.nonzero(bits)[0][:cnt] + b).astype(np.uint64)
            counts.append(cnt)
            if cnt:
                ch, est = O.select_per_input(n, m, space.cost, occ, queued, slots, mean, 1, members)
                d = [(ch // m ** (n - 1 - a)) % m for a in range(n)]
                c = 0.0
                for x in d:
                    c += float(space.cost[x])
                best_e.append(est)
                best_c.append(c)
                best_i.append(ch)
            else:
                best_e.append(np.inf)
                best_c.append(np.inf)
                best_i.append(0)
        rec = PL.pack_records(counts, best_e, best_c, best_i)
        # the sharded path's one collective, on CPU tensors over gloo
        import torch
        g = PL.exchange_records(torch.from_numpy(rec.view(np.int64).copy()), world)
        assert tuple(g.shape) == (world, R, PL.REC_WORDS)
        gathered = g.numpy().view(np.uint64)
        assert np.array_equal(gathered, PL.all_gather_records(rec))
        total, before, (ge, gc, gi) = PL.merge_records(gathered, rank)
        # the whole-space oracle
        ok = True
        for r in range(R):
            cnt, words = O.enumerate_bitmap(tb, O.Router(0, 0, 0, 0, 0), r, 0, space.size)
            bits = np.unpackbits(words.view(np.uint8), bitorder="little")
            members = np.nonzero(bits)[0][:cnt].astype(np.uint64)
            ok &= int(total[r]) == cnt
            ok &= int(before[r]) == int(np.sum(members < b))
            ch, est = O.select_per_input(n, m, space.cost, occ, queued, slots, mean, 1, members)
            ok &= int(gi[r]) == ch and float(ge[r]) == est
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_sharded_merge_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]


def test_bench_spawns_one_rank_per_gpu():
    """`bench.py --gpus N` without a launcher re-executes itself under
    torchrun (one process per GPU, rendezvous on 127.0.0.1); the ranks join
    one process group and rank 0 reports n_gpus = N."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--spawn-selftest"],
                         capture_output=True, text=True, timeout=240, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["ranks_joined"] == 2 and line["launcher"] == "torchrun"
