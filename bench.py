#!/usr/bin/env python
"""bench.py -- Aragog hot paths on B200.

Headline (BASELINE.json metric "configs routed/sec ..."): enumerate-mode
routing of BASELINE config 2 -- a 5-stage chain x 8 model tiers (32,768
configurations per request), a 10k-request batch per GPU, oracle router --
through the C ABI (libaragog_b200.so).  One step = route one batch:
score every configuration, scan, stream-compact the accurate set.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one process per GPU; requests are sharded (each
rank routes its own 10k requests, no data-path collective: weak scaling);
the timed region is bracketed by barrier + synchronize and the max over ranks
is taken.  `--impl reference` times the reference's own CPU implementation
(oracle/_ref/ref_bench, compiled from /root/reference) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_AGENTS, N_TIERS, REQUESTS_PER_GPU, SEED = 5, 8, 10_000, 1
METRIC = "configs routed/sec"
UNIT = "configs/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
CPU_SAMPLE_REQUESTS = 1000


def workload_config(n_gpus):
    return {"workload": f"config2: chain {N_AGENTS} stages x {N_TIERS} tiers "
                        f"({N_TIERS ** N_AGENTS} configs/request), enumerate mode, oracle router",
            "requests_per_gpu": REQUESTS_PER_GPU, "global_requests": REQUESTS_PER_GPU * n_gpus,
            "configs_per_request": N_TIERS ** N_AGENTS, "seed": SEED,
            "accuracy_gen": "AccuracyGenParams{} (easy .6 / medium .3 / hard .1, base .5)",
            "parallelism": f"request-sharded x{n_gpus}",
            "l2": "flushed before every timed step (256 MiB write)"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return p["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)["kernels"][kernel]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def cpu_baseline(sample=CPU_SAMPLE_REQUESTS, threads=None):
    """The reference's own enumerate-mode loop on the host cores (ref_bench)."""
    threads = threads or os.cpu_count()
    if os.path.exists(REF_BENCH):
        out = subprocess.run([REF_BENCH, "route", str(N_AGENTS), str(N_TIERS), str(sample),
                              "oracle", str(threads), str(SEED)], capture_output=True, text=True,
                             check=True).stdout
        r = json.loads(out.strip().splitlines()[-1])
        return {"value": r["configs_per_s"], "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"first {sample} requests of config 2 "
                          f"({sample * N_TIERS ** N_AGENTS:.3g} configs), reference "
                          "at_index+OracleRouter::evaluate loop under parallel_for"}
    # port: the C restatement, single thread, bounded sample
    from oracle import oracle as O
    import paper_2511_20975_b200 as P
    space = P.ConfigSpace.chain(N_AGENTS, N_TIERS)
    b = P.AccuracyBatch.generate(space, P.GenParams(), 50, SEED)
    tb = O.TruthBatch(N_AGENTS, N_TIERS, [b.seeds_of(r) for r in range(50)],
                      [b.removed_of(r) for r in range(50)], b.request_ids)
    t0 = time.perf_counter()
    for r in range(50):
        O.enumerate_bitmap(tb, O.Router(O.ORACLE, 0, 0, 0, 0), r, 0, space.size)
    dt = time.perf_counter() - t0
    return {"value": 50 * space.size / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": "50 requests of config 2, C oracle restatement"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count()
    if not os.path.exists(REF_BENCH):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_bench not built"}))
        return
    times, vals = [], []
    for i in range(args.warmup + args.steps):
        base = cpu_baseline(CPU_SAMPLE_REQUESTS, threads)
        if i >= args.warmup:
            vals.append(base["value"])
    v = statistics.median(vals)
    ms = CPU_SAMPLE_REQUESTS * N_TIERS ** N_AGENTS / v * 1e3
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "impl": "reference", "config": workload_config(1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{CPU_SAMPLE_REQUESTS} requests of config 2 per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_ours(args):
    import torch

    import paper_2511_20975_b200 as P

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev_t = torch.device("cuda", local)

    space = P.ConfigSpace.chain(N_AGENTS, N_TIERS)
    batch = P.AccuracyBatch.generate(space, P.GenParams(), REQUESTS_PER_GPU, SEED,
                                     first_id=rank * REQUESTS_PER_GPU)
    stream = torch.cuda.current_stream(dev_t)
    dev = P.Device(space, local, stream)
    truth = batch.to_device(dev_t)
    router = P.OracleRouter()
    S = space.size
    # capacity from a first pass (members are deterministic per batch)
    probe = dev.route_enumerate(truth, router, compact=False)
    torch.cuda.synchronize()
    total_members = int(probe.offsets[-1])
    out = dev.alloc_route(REQUESTS_PER_GPU, 0, S, total_members)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev_t)

    def step():
        dev.route_enumerate(truth, router, out=out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region (value) + live per-kernel profile
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = Clocks(local)
    launches0 = dev.launch_count
    barrier()
    dev.profile_begin()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    kprof = dev.profile_end()
    barrier()
    clk = clocks.stop()
    launches = dev.launch_count - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev_t)
    if ws > 1:
        torch.distributed.all_reduce(tot_ms, op=torch.distributed.ReduceOp.MAX)
    tot_ms = float(tot_ms.item())
    configs_total = args.steps * REQUESTS_PER_GPU * S * ws
    value = configs_total / (tot_ms / 1e3)

    # ---- e2e through the host-buffer C ABI call (H2D + D2H inside the region)
    hb_counts = np.zeros(REQUESTS_PER_GPU, np.uint64)
    hb_offsets = np.zeros(REQUESTS_PER_GPU + 1, np.uint64)
    import ctypes as C
    pinned = C.c_void_p()
    P._capi.check(P.lib().ag_host_alloc(C.c_size_t(4 * total_members), C.byref(pinned)))
    hb_idx = np.ctypeslib.as_array((C.c_uint32 * total_members).from_address(pinned.value))
    e2e_steps = max(1, min(args.steps, 5))
    dev.route_enumerate_host(batch, router, indices=hb_idx, counts=hb_counts, offsets=hb_offsets)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dev.route_enumerate_host(batch, router, indices=hb_idx, counts=hb_counts,
                                 offsets=hb_offsets)
    barrier()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev_t)
    if ws > 1:
        torch.distributed.all_reduce(e2e_s, op=torch.distributed.ReduceOp.MAX)
    e2e_value = e2e_steps * REQUESTS_PER_GPU * S * ws / float(e2e_s.item())
    h2d = (batch.request_ids.nbytes + batch.seed_ptr.nbytes + batch.seeds.nbytes +
           batch.removed_ptr.nbytes + batch.removed.nbytes)
    d2h = hb_counts.nbytes + hb_offsets.nbytes + 4 * total_members
    ok = int(hb_offsets[-1]) == total_members
    P.lib().ag_host_free(pinned)

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (algorithmic bytes / avg duration)
    hbm, peak_src = peaks()
    W = (S + 31) // 32
    bitmap_bytes = REQUESTS_PER_GPU * W * 4
    algo = {"k_route_score": bitmap_bytes,                       # bitmap write
            "k_route_compact": bitmap_bytes + 4 * total_members,  # bitmap read + index write
            "k_chunk_scan": REQUESTS_PER_GPU * (W // 32) * 12 + 8 * REQUESTS_PER_GPU,
            "k_request_scan": 16 * REQUESTS_PER_GPU}
    dom = max(kprof, key=lambda k: kprof[k][0])
    dom_ms = kprof[dom][0] / kprof[dom][1]
    achieved = algo.get(dom, 0) / (dom_ms / 1e3) / 1e9
    kernel_share = {k: round(v[0] / sum(x[0] for x in kprof.values()), 4) for k, v in kprof.items()}
    path_bytes = bitmap_bytes + 4 * total_members  # per step output
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "impl": "ours", "config": workload_config(ws),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "members_ok": ok,
                "path": "ag_route_enumerate_host (pinned host indices)"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "peak_source": peak_src,
                     "traffic": ncu_traffic(dom),
                     "algorithmic_bytes_per_launch": algo.get(dom, 0),
                     "avg_launch_ms": dom_ms},
        "path_roofline": {"bytes_per_step": path_bytes,
                          "achieved_gbs": path_bytes / (tot_ms / args.steps / 1e3) / 1e9},
        "kernel_share": kernel_share,
        "members_per_step": total_members,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
