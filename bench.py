#!/usr/bin/env python
"""bench.py -- Aragog's two hot paths on B200, through the C ABI.

Headline (BASELINE.json metric "configs routed/sec and p50/p99 per-stage
scheduling latency"):

  * routing, BASELINE config 2: enumerate-mode routing of a 5-stage chain x 8
    model tiers (32,768 configurations per request), a 10k-request batch per
    GPU, oracle router.  One step = route one batch: score every
    configuration, scan, stream-compact the accurate set.  `value` is
    configurations routed per second over all GPUs (inputs resident in HBM);
    `e2e` is the same through the host-buffer call with copies included.
  * per-stage scheduling, BASELINE config 3: 10k in-flight requests resident
    on the GPU, 8 pools x 32 slots, free slots per round drawn from {1, 8, 64},
    beam width 4; p50/p99 of the decision latency of ag_sched_round (host
    wall time inside the C ABI call: upload of pending updates, the round
    kernel, download of the assignment).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one process per GPU; requests are sharded (each
rank routes its own 10k requests, no data-path collective: weak scaling); the
timed region is bracketed by barrier + synchronize and the max over ranks is
taken.  Scheduling is a per-GPU latency (replicas only, reported by rank 0).
`--impl reference` times the reference's own CPU implementation
(oracle/_ref/ref_bench, compiled unmodified from /root/reference).
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
SCHED_INFLIGHT, SCHED_BEAM = 10_000, 4


def workload_config(n_gpus):
    return {"workload": f"config2: chain {N_AGENTS} stages x {N_TIERS} tiers "
                        f"({N_TIERS ** N_AGENTS} configs/request), enumerate mode, oracle router",
            "requests_per_gpu": REQUESTS_PER_GPU, "global_requests": REQUESTS_PER_GPU * n_gpus,
            "configs_per_request": N_TIERS ** N_AGENTS, "seed": SEED,
            "accuracy_gen": "AccuracyGenParams{} (easy .6 / medium .3 / hard .1, base .5)",
            "parallelism": f"request-sharded x{n_gpus}",
            "l2": "flushed before every timed step (256 MiB write)",
            "sched_workload": f"config3: {SCHED_INFLIGHT} in-flight requests (chain 5x8, viable sets "
                              "from chain-mode predict), 8 pools x 32 slots, free slots "
                              f"{{1,8,64}} per round, beam {SCHED_BEAM}"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # multi-rank logic check on a one-GPU box (tests only): every rank on
    # cuda:0, gloo for the collectives (NCCL refuses two ranks on one device)
    if os.environ.get("AG_BENCH_ONE_DEVICE") == "1":
        local = 0
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling (clocks and throttle reasons) while work runs."""

    FIELDS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        self.p.wait()
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        finally:
            os.unlink(self.path)
        sm, mx, reasons = [], None, set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(self.FIELDS, r[3:7]):
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


def ref_route(sample, threads):
    out = subprocess.run([REF_BENCH, "route", str(N_AGENTS), str(N_TIERS), str(sample), "oracle",
                          str(threads), str(SEED)], capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def ref_sched(rounds, beam=SCHED_BEAM, exhaustive=False):
    out = subprocess.run([REF_BENCH, "sched", str(SCHED_INFLIGHT), str(beam), str(rounds),
                          str(SEED), "1" if exhaustive else "0"],
                         capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


SELECT_CPU_SAMPLE = {"exhaustive": 1000, "viable": REQUESTS_PER_GPU}


def ref_select(sets, requests, threads):
    out = subprocess.run([REF_BENCH, "select", str(N_AGENTS), str(N_TIERS), str(requests), str(threads),
                          str(SEED), sets], capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def select_load(m):
    """The select leg's load context (ref_bench select): occupancy 4,
    queued_ahead i % 3, 8 slots, ServiceTimeModel{mu -0.3 + 0.35 i, sigma
    0.25, floor 0.05}::mean computed with the C library's exp, as the
    reference does (engine.cpp:62-65)."""
    import math

    mean = [0.05 + math.exp((-0.3 + 0.35 * i) + 0.5 * 0.25 * 0.25) for i in range(m)]
    return [4] * m, [i % 3 for i in range(m)], [8] * m, mean


def select_digest(chosen, est, n):
    """ref_bench select's digest: D = mix({D, index, estimate bits}) over
    the first n requests."""
    from paper_2511_20975_b200 import workloads as W

    bits = np.asarray(est[:n], np.float64).view(np.uint64)
    d = 0x5EED
    for i in range(n):
        d = W.mix(d, int(chosen[i]), int(bits[i]))
    return f"{d:016x}"


# config-3 variants beside the headline (B = 4, predictor sets): the other
# beam width SURVEY.md §8(d) names, and exhaustive viable sets (the full
# accurate set per request, 13.5k configurations on average)
SCHED_VARIANTS = {"beam1": {"beam": 1, "exhaustive": False, "rounds": 300, "ref_rounds": 310},
                  "exhaustive": {"beam": SCHED_BEAM, "exhaustive": True, "rounds": 100,
                                 "ref_rounds": 6}}


def absorb_peak():
    """Measured rng::mix absorb steps/s of this GPU (scripts/ubench/mix_peak),
    the integer-issue ceiling of the noisy router; None if not built."""
    exe = os.path.join(ROOT, "scripts", "ubench", "mix_peak")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
        return float(json.loads(out.strip().splitlines()[-1])["absorbs_per_s"])
    except (OSError, ValueError, KeyError, IndexError, subprocess.TimeoutExpired):
        return None


def ubench_bw():
    """Measured HBM-by-direction and PCIe ceilings (scripts/ubench/bw)."""
    exe = os.path.join(ROOT, "scripts", "ubench", "bw")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
        return json.loads(out.strip().splitlines()[-1])
    except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
        return None


def host_info():
    """CPU model, cores, compiler of the reference build."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        gxx = subprocess.run(["g++", "--version"], capture_output=True, text=True).stdout.splitlines()[0]
    except (OSError, IndexError):
        gxx = "unknown"
    return {"cpu": model, "nproc": os.cpu_count(), "compiler": gxx,
            "flags": "-std=c++20 -O2 (no -march: no FMA contraction, as the reference)"}


def cpu_baseline(sample=CPU_SAMPLE_REQUESTS, threads=None):
    """The reference's own enumerate-mode loop on the host cores (ref_bench),
    plus one core, the chain-mode predictor and the host description."""
    threads = threads or os.cpu_count()
    if os.path.exists(REF_BENCH):
        r = ref_route(sample, threads)
        one = ref_route(max(sample // 10, 1), 1)
        out = subprocess.run([REF_BENCH, "predict", str(N_AGENTS), str(N_TIERS), "2000", "oracle",
                              str(threads), str(SEED)], capture_output=True, text=True,
                             check=True).stdout
        pr = json.loads(out.strip().splitlines()[-1])
        return {"value": r["configs_per_s"], "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"first {sample} requests of config 2 "
                          f"({sample * N_TIERS ** N_AGENTS:.3g} configs), reference "
                          "at_index+OracleRouter::evaluate loop under parallel_for",
                "one_core": {"value": one["configs_per_s"], "unit": UNIT,
                             "sample": f"{max(sample // 10, 1)} requests"},
                "chain_mode": {"value": pr["requests_per_s"], "unit": "requests/s",
                               "cores": threads, "sample": "2000 requests, predict(inf)"},
                "host": host_info()}
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
    vals = []
    for i in range(args.warmup + args.steps):
        r = ref_route(CPU_SAMPLE_REQUESTS, threads)
        if i >= args.warmup:
            vals.append(r["configs_per_s"])
    v = statistics.median(vals)
    ms = CPU_SAMPLE_REQUESTS * N_TIERS ** N_AGENTS / v * 1e3
    sched = ref_sched(args.sched_rounds + args.sched_warmup)
    variants = {}
    if not args.no_sched_variants:
        for name, sv in SCHED_VARIANTS.items():
            r = ref_sched(sv["ref_rounds"], sv["beam"], sv["exhaustive"])
            variants[name] = {"beam": sv["beam"], "exhaustive": sv["exhaustive"],
                              "p50_us": r["p50_us"], "p99_us": r["p99_us"], "rounds": r["rounds"]}
    select = {}
    if not args.no_select:
        for sets in ("exhaustive", "viable"):
            r = ref_select(sets, SELECT_CPU_SAMPLE[sets], threads)
            select[sets] = {"configs_costed_per_s": r["configs_costed_per_s"],
                            "us_per_batch": r["us_per_request"] * REQUESTS_PER_GPU,
                            "sample": f"first {SELECT_CPU_SAMPLE[sets]} requests", "cores": threads}
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "impl": "reference", "config": workload_config(1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{CPU_SAMPLE_REQUESTS} requests of config 2 per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "sched": {"p50_us": sched["p50_us"], "p99_us": sched["p99_us"],
                      "mean_us": sched["mean_us"], "rounds": sched["rounds"], "cores": 1,
                      "decision_hash": sched["hash"], "variants": variants,
                      "what": "beam_schedule per round, reference C++ on one core"},
            "select": select}
    print(json.dumps(line))


def run_sched(P, W, dev, args, rounds=None, beam=SCHED_BEAM, exhaustive=False):
    """Config 3 on this GPU: p50/p99 of the C-ABI round latency."""
    rounds = args.sched_rounds if rounds is None else rounds
    c3 = W.Config3(dev, inflight=SCHED_INFLIGHT, rounds=rounds + args.sched_warmup,
                   seed=SEED, beam=beam, exhaustive=exhaustive)
    dev_us, capi_us, free = [], [], []
    weights = list(c3.space.slot_throughput)

    def on_round(rd, a):
        if rd >= args.sched_warmup:
            t = c3.sess.round_timing()
            dev_us.append(float(t.sum()))
            capi_us.append(c3.sess.last_round_us())
            free.append(W.config3_engines(rd, SEED, weights)[1])

    _, h, assigned = c3.run(on_round=on_round)
    capi = np.asarray(capi_us)
    disp = np.asarray(c3.dispatch_us[args.sched_warmup:])
    both = capi + disp[: len(capi)]
    devt = np.asarray(dev_us)
    free = np.asarray(free)
    by_free = {}
    for f in sorted(set(free.tolist())):
        sel = capi[free == f]
        by_free[str(f)] = {"rounds": int(sel.size), "p50_us": float(np.percentile(sel, 50)),
                           "p99_us": float(np.percentile(sel, 99))}
    return {"p50_us": float(np.percentile(capi, 50)), "p99_us": float(np.percentile(capi, 99)),
            "mean_us": float(capi.mean()),
            "device_p50_us": float(np.percentile(devt, 50)),
            "device_p99_us": float(np.percentile(devt, 99)),
            "dispatch_p50_us": float(np.percentile(disp, 50)), "dispatch_p99_us": float(np.percentile(disp, 99)),
            "round_plus_dispatch_p50_us": float(np.percentile(both, 50)),
            "round_plus_dispatch_p99_us": float(np.percentile(both, 99)),
            "rounds": len(capi), "warmup_rounds": args.sched_warmup, "assigned": int(assigned),
            "by_free_slots": by_free,
            "decision_hash": f"{h:016x}",
            "what": "ag_sched_round wall time inside the C ABI (update upload + round kernel + "
                    "assignment download); device = the round kernel alone"}


def run_select(P, dev, sets, members, offsets, n_members, stream, flush, barrier, with_ref, bitmap=None,
               counts=None):
    """The per-stage re-cost + argmin of config 3:
    select_per_input_config(set, space, kPerInputRuntimeCost, &ctx) for all
    10k requests of the batch, device-resident member CSR, CUDA-event timed
    (µs per 10k-request batch), HBM roofline at 4 B read per member; the
    reference (ref_bench select) on all host cores beside it, and the digest
    of (chosen, estimate) over its sample equal to the reference's."""
    import torch

    m = dev.space.m
    occ, queued, slots, mean = select_load(m)
    load = P.RuntimeCostContext(occ, queued, slots, mean)
    R = REQUESTS_PER_GPU
    for _ in range(3):
        ch, est = P.select_per_input(dev, members, offsets, P.PER_INPUT_RUNTIME_COST, load,
                                     check_errors=False)
    dev.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    barrier()
    dev.profile_begin()
    for i in range(10):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        ch, est = P.select_per_input(dev, members, offsets, P.PER_INPUT_RUNTIME_COST, load,
                                     check_errors=False)
        ev[i][1].record(stream)
    kprof = dev.profile_end()
    dev.synchronize()
    ms = statistics.median([a.elapsed_time(b) for a, b in ev])
    kms = kprof["k_cost_argmin"][0] / 10 if "k_cost_argmin" in kprof else ms
    hbm, psrc = peaks()
    out = {"workload": f"config3 re-cost + argmin: select_per_input_config(kPerInputRuntimeCost) over "
                       f"the {sets} sets of {R} config-2 requests ({n_members} members), load context "
                       "of ref_bench select",
           "us_per_batch": ms * 1e3, "configs_costed_per_s": n_members / (ms / 1e3),
           "launches_per_batch": 4,
           "roofline": {"bound": "hbm", "kernel": "k_cost_plan/prefix/tasks/reduce",
                        "achieved": 4.0 * n_members / (kms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                        "frac": 4.0 * n_members / (kms / 1e3) / 1e9 / hbm, "peak_source": psrc,
                        "algorithmic_bytes_per_launch": 4 * n_members}}
    if bitmap is not None:
        # the same selection straight from the verdict bitmap (ag_select_bitmap)
        S = dev.space.size
        for _ in range(3):
            bch, best = P.select_bitmap(dev, bitmap, counts, 0, S, P.PER_INPUT_RUNTIME_COST, load,
                                        check_errors=False)
        dev.synchronize()
        barrier()
        dev.profile_begin()
        for i in range(10):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            bch, best = P.select_bitmap(dev, bitmap, counts, 0, S, P.PER_INPUT_RUNTIME_COST, load,
                                        check_errors=False)
            ev[i][1].record(stream)
        bprof = dev.profile_end()
        dev.synchronize()
        bms = statistics.median([a.elapsed_time(b) for a, b in ev])
        bkms = bprof["k_cost_argmin"][0] / 10 if "k_cost_argmin" in bprof else bms
        bbytes = R * ((S + 31) // 32) * 4
        out["bitmap_path"] = {
            "us_per_batch": bms * 1e3, "configs_costed_per_s": n_members / (bms / 1e3), "launches_per_batch": 3,
            "same_as_member_path": bool(torch.equal(bch, ch) and torch.equal(best, est)),
            "roofline": {"bound": "hbm", "kernel": "k_bm_prefix/eval/reduce",
                         "achieved": bbytes / (bkms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": bbytes / (bkms / 1e3) / 1e9 / hbm, "peak_source": psrc,
                         "algorithmic_bytes_per_launch": bbytes}}
    if with_ref and os.path.exists(REF_BENCH):
        n = SELECT_CPU_SAMPLE[sets]
        ref = ref_select(sets, n, os.cpu_count())
        chn = ch.cpu().numpy().view(np.uint32)
        estn = est.cpu().numpy()
        out["reference"] = {"configs_costed_per_s": ref["configs_costed_per_s"],
                            "us_per_batch": ref["us_per_request"] * R, "cores": ref["threads"],
                            "sample": f"first {n} requests", "kind": "reference"}
        out["digest_match"] = select_digest(chn, estn, n) == ref["digest"]
    return out


def run_deep(P, args, ws, rank, local, barrier):
    """Config 4: 8 stages x 12 tiers (4.3e8 configurations per request), 16
    requests, the canonical-index space split contiguously across the ranks
    (strong scaling), then one all-gather of per-shard records (counts and
    the runtime-cost minimum) -- paper_2511_20975_b200.parallel."""
    import torch

    from paper_2511_20975_b200 import parallel as PL

    n, m, R = 8, 12, 16
    dev_t = torch.device("cuda", local)
    space = P.ConfigSpace.chain(n, m)
    dev = P.Device(space, local, torch.cuda.current_stream(dev_t))
    batch = P.AccuracyBatch.generate(space, P.GenParams(), R, SEED)
    truth = batch.to_device(dev_t)
    router = P.OracleRouter()
    begin, end = PL.shard_range(space.size, rank, ws)
    probe = dev.route_enumerate(truth, router, begin, end, compact=False)
    torch.cuda.synchronize()
    cap = int(probe.offsets[-1])
    out = dev.alloc_route(R, begin, end, cap, bitmap=True)  # the argmin reads the verdict bitmap
    mean = [0.05 + float(np.exp(-0.3 + 0.35 * i + 0.5 * 0.25 * 0.25)) for i in range(m)]
    load = P.RuntimeCostContext([4] * m, [i % 3 for i in range(m)], [8] * m, mean)
    times = []
    steps = max(2, min(args.steps, 5))
    stream = torch.cuda.current_stream(dev_t)
    kprof = None
    for i in range(1 + steps):
        barrier()
        torch.cuda.synchronize()
        if i == steps:
            dev.profile_begin()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res, total, before, best = PL.route_space_sharded(dev, truth, router, rank, ws, load, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        if i == steps:
            kprof = dev.profile_end()
        barrier()
        if i:
            times.append(e0.elapsed_time(e1) / 1e3)
    dt = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev_t)
    if ws > 1:
        torch.distributed.all_reduce(dt, op=torch.distributed.ReduceOp.MAX)
    dt = float(dt.item())
    configs = R * space.size
    del out, res, probe
    torch.cuda.empty_cache()
    return {"workload": "config4: chain 8 x 12 tiers (4.3e8 configs/request), 16 requests, "
                        f"canonical-index space sharded over {ws} GPU(s), oracle router, "
                        "enumerate + compact + runtime-cost argmin from the verdict bitmap + all-gather of 32-byte "
                        "per-shard records",
            "configs_per_s": configs / dt, "ms_per_step": dt * 1e3, "scaling": "strong",
            "members": int(total.sum()), "n_gpus": ws,
            "kernel_ms": {k: v[0] / v[1] for k, v in (kprof or {}).items()},
            "timing": "CUDA events on the launching stream around the whole sharded step "
                      "(host round trips and the NCCL all-gather included), max over ranks, "
                      "median of steps"}


INTEG = os.path.join(ROOT, "integration", "_build")
C5_RATES = (0.5, 1.5, 2.5, 3.5)


def run_config5(horizon=240.0):
    """Config 5: the reference simulator (run_simulation, reference.json) over
    the shipped sweep rates in horizon mode, built twice from the unmodified
    sources -- plain, and relinked with the GPU adapter (predict, beam
    rounds, per-input selection on the B200; integration/Makefile).  Reports
    wall-clock scheduling rounds/s of both builds and whether the JSONL traces
    are byte-identical."""
    ref_bin, gpu_bin = os.path.join(INTEG, "sim_trace_ref"), os.path.join(INTEG, "sim_trace_gpu")
    scen = os.path.join(INTEG, "proj", "scenarios", "reference.json")
    if not (os.path.exists(ref_bin) and os.path.exists(gpu_bin) and os.path.exists(scen)):
        return None
    def sweep(scenario, rates, hz, td):
        rows, ok = [], True
        for rate in rates:
            row = {"rate": rate}
            outs = []
            for kind, b in (("reference", ref_bin), ("gpu", gpu_bin)):
                out = os.path.join(td, f"{kind}_{rate}.jsonl")
                r = subprocess.run([b, scenario, "aragog", out, "--horizon", str(hz), "--rate",
                                    str(rate)], capture_output=True, text=True, check=True)
                j = json.loads(r.stdout.strip().splitlines()[-1])
                row[kind] = {"rounds": j["rounds"], "requests": j["requests"],
                             "wall_s": j["wall_s"], "rounds_per_s": j["rounds_per_s"],
                             "gpu_launches": j["gpu_launches"]}
                outs.append(open(out, "rb").read())
            row["trace_identical"] = outs[0] == outs[1]
            ok &= row["trace_identical"]
            rows.append(row)
        return rows, ok

    with tempfile.TemporaryDirectory() as td:
        pts, same = sweep(scen, C5_RATES, horizon, td)
    # decompose.json (the diamond workflow: plan -> {search, math} -> synth)
    # over its own shipped sweep rates and horizon
    decompose = None
    dscen = os.path.join(INTEG, "proj", "scenarios", "decompose.json")
    if os.path.exists(dscen):
        dsw = json.load(open(dscen)).get("sweep", {})
        with tempfile.TemporaryDirectory() as td:
            dpts, dsame = sweep(dscen, dsw.get("rates", [1.0]), dsw.get("horizon", 180), td)
        decompose = {"points": dpts, "traces_identical": dsame}
        same &= dsame
    # BASELINE scale: a 5-stage chain x 8 tiers scenario (the config-2 space)
    # with ~500-960 requests queued per round, drained
    scale = None
    with tempfile.TemporaryDirectory() as td:
        sc = {"name": "chain5x8", "seed": 1,
              "workflow": {"agents": [f"a{i}" for i in range(5)],
                           "edges": [[f"a{i}", f"a{i + 1}"] for i in range(4)]},
              "models": [{"name": f"m{i}", "cost": 1.5 ** i, "slot_throughput": 8.0 / 1.5 ** i}
                         for i in range(8)],
              "engines": [{"model": f"m{i}", "slots": 32,
                           "service": {"mu": -0.3 + 0.35 * i, "sigma": 0.25, "floor": 0.05}}
                          for i in range(8)],
              "router": {"kind": "oracle", "eval_latency": 0.002},
              "predictor": {"min_budget": 0.12, "ema_alpha": 0.2, "router_lanes": 16},
              "accuracy": {"p_easy": 0.6, "p_medium": 0.3, "p_hard": 0.1, "easy_base_prob": 0.5},
              "workload": {"arrival_rate": 60.0, "num_requests": 1200, "horizon": 240,
                           "per_workflow_sample": 256},
              "scheduler": {"beam_width": 4},
              "sweep": {"rates": [60.0], "seeds": [1], "horizon": 60},
              "metrics": {"sample_interval": 0.5}}
        sp = os.path.join(td, "chain5x8.json")
        json.dump(sc, open(sp, "w"))
        row, outs = {"scenario": "chain5x8 (5 stages x 8 tiers, 8 pools x 32 slots, 60 req/s, "
                                 "1200 requests, drain)"}, []
        for kind, b in (("reference", ref_bin), ("gpu", gpu_bin)):
            out = os.path.join(td, f"{kind}_scale.jsonl")
            r = subprocess.run([b, sp, "aragog", out, "--requests", "1200"], capture_output=True,
                               text=True, check=True)
            j = json.loads(r.stdout.strip().splitlines()[-1])
            row[kind] = {"rounds": j["rounds"], "pairs": j["pairs"], "wall_s": j["wall_s"],
                         "rounds_per_s": j["rounds_per_s"], "gpu_launches": j["gpu_launches"]}
            outs.append(open(out, "rb").read())
        row["trace_identical"] = outs[0] == outs[1]
        same &= row["trace_identical"]
        scale = row
    return {"workload": f"config5: reference.json under run_simulation, horizon {horizon:g} s, "
                        f"aragog policy, rates {list(C5_RATES)} req/s, and decompose.json over its "
                        "own sweep; reference build vs the same sources relinked with the GPU "
                        "adapter; plus a 5x8 scenario at BASELINE scale",
            "traces_identical": same, "points": pts, "scale": scale, "decompose": decompose,
            "note": "single-request decisions through the C ABI: each predict / round is one "
                    "launch + synchronisation, so tiny queues are launch-latency bound"}


def run_config1():
    """Config 1: the smallest bundled scenario,
    reference.json (3 stages x 3 tiers), 1,000 requests, seed 1, policy
    aragog, drain mode -- and the 3 x 4 variant adding tier "xl" (cost 9.0,
    weight 0.4, 4 slots, service mu 1.6, sigma 0.25, floor 0.05) -- through
    the reference's CPU router + scheduler (sim_trace_ref) and the same
    sources relinked with the GPU adapter (sim_trace_gpu): wall time of the
    run and trace identity."""
    ref_bin, gpu_bin = os.path.join(INTEG, "sim_trace_ref"), os.path.join(INTEG, "sim_trace_gpu")
    scen = os.path.join(INTEG, "proj", "scenarios", "reference.json")
    if not (os.path.exists(ref_bin) and os.path.exists(gpu_bin) and os.path.exists(scen)):
        return None
    pts = []
    with tempfile.TemporaryDirectory() as td:
        base = json.load(open(scen))
        xl = json.loads(json.dumps(base))
        xl["name"] = "reference_xl"
        xl["models"].append({"name": "xl", "cost": 9.0, "slot_throughput": 0.4})
        xl["engines"].append({"model": "xl", "slots": 4, "service": {"mu": 1.6, "sigma": 0.25, "floor": 0.05}})
        xl_path = os.path.join(td, "reference_xl.json")
        json.dump(xl, open(xl_path, "w"))
        for name, path in (("reference 3x3", scen), ("reference_xl 3x4", xl_path)):
            row = {"name": name}
            outs = []
            for kind, b in (("reference", ref_bin), ("gpu", gpu_bin)):
                out = os.path.join(td, f"{kind}_{len(pts)}.jsonl")
                r = subprocess.run([b, path, "aragog", out, "--requests", "1000", "--seed", "1"],
                                   capture_output=True, text=True, check=True)
                j = json.loads(r.stdout.strip().splitlines()[-1])
                row[kind] = {"rounds": j["rounds"], "requests": j["requests"], "wall_s": j["wall_s"],
                             "rounds_per_s": j["rounds_per_s"], "gpu_launches": j["gpu_launches"]}
                outs.append(open(out, "rb").read())
            row["identical"] = outs[0] == outs[1]
            pts.append(row)
    return {"workload": "config1: reference.json (3x3) and its 3x4 xl variant, 1000 requests, seed 1, "
                        "aragog policy, drain mode; reference build vs the GPU-adapter build",
            "points": pts}


def run_ours(args):
    import torch

    import paper_2511_20975_b200 as P
    from paper_2511_20975_b200 import workloads as W

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if os.environ.get("AG_BENCH_ONE_DEVICE") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev_t = torch.device("cuda", local)
    clocks = Clocks(local)

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
    out = dev.alloc_route(REQUESTS_PER_GPU, 0, S, total_members, bitmap=True)
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
    launches0 = dev.launch_count
    barrier()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    barrier()
    launches = dev.launch_count - launches0
    # the live per-kernel profile (CUDA events around every launch) on extra
    # steps: events between the kernels would serialise their programmatic
    # dependent launches inside the timed steps
    dev.profile_begin()
    for i in range(max(3, min(args.steps, 10))):
        flush.fill_(i & 0xFF)
        step()
    kprof = dev.profile_end()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev_t)
    if ws > 1:
        torch.distributed.all_reduce(tot_ms, op=torch.distributed.ReduceOp.MAX)
    tot_ms = float(tot_ms.item())
    configs_total = args.steps * REQUESTS_PER_GPU * S * ws
    value = configs_total / (tot_ms / 1e3)
    # parity spot check of this run's output against its own bitmap count
    ok_counts = int(out["offsets"][-1]) == total_members

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
    e2e_ok = int(hb_offsets[-1]) == total_members
    P.lib().ag_host_free(pinned)
    # the e2e ceiling: the step's PCIe bytes at the measured pinned copy rates
    bw = ubench_bw() if rank == 0 and not args.no_ubench else None
    e2e_roof = None
    if bw and bw.get("pcie_d2h_gbs"):
        t_min = d2h / (bw["pcie_d2h_gbs"] * 1e9) + h2d / (bw["pcie_h2d_gbs"] * 1e9)
        e2e_roof = {"bound": "pcie", "bytes_per_step": int(h2d + d2h),
                    "floor_ms_per_step": t_min * 1e3,
                    "achieved_ms_per_step": float(e2e_s.item()) / e2e_steps * 1e3,
                    "frac": t_min / (float(e2e_s.item()) / e2e_steps),
                    "peak_source": "scripts/ubench/bw (pinned cudaMemcpyAsync, measured live)",
                    "ubench": bw}

    # chain mode (ConfigPredictor::predict, the reference's routing call):
    # the same 10k requests, unbounded budget and the 0.002 s evaluation charge
    chain = None
    if not args.no_chain:
        pred = P.ConfigPredictor(dev)
        crouter = P.OracleRouter(0.002)
        for _ in range(2):
            pred.predict_batch(truth, crouter)
        cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(5)]
        barrier()
        for i in range(5):
            flush.fill_(i & 0xFF)
            cev[i][0].record(stream)
            cres = pred.predict_batch(truth, crouter)
            cev[i][1].record(stream)
        barrier()
        cms = statistics.median([x.elapsed_time(y) for x, y in cev])
        chain = {"workload": "config2 requests through ConfigPredictor::predict (chain plan, "
                             "binary search, verification; budget inf)",
                 "requests_per_s": REQUESTS_PER_GPU / (cms / 1e3), "ms_per_batch": cms,
                 "evaluations_per_request": float((cres.search_evals + cres.verify_evals)
                                                  .double().mean().item()),
                 "viable_per_request": float(cres.n_viable.double().mean().item())}
        csel = None
        if not args.no_select:
            nv = cres.n_viable.to(torch.int64)
            cmask = torch.arange(cres.viable.shape[1], device=dev_t)[None, :] < nv[:, None]
            cmem = cres.viable[cmask].contiguous()
            coffs = torch.zeros(REQUESTS_PER_GPU + 1, dtype=torch.int64, device=dev_t)
            coffs[1:] = torch.cumsum(nv, 0)
            csel = run_select(P, dev, "viable", cmem, coffs, int(coffs[-1]), stream, flush, barrier,
                              rank == 0 and not args.no_cpu_baseline)
            del cmem, coffs, cmask
        del pred, cres
    select = None
    if not args.no_select:
        select = run_select(P, dev, "exhaustive", out["indices"], out["offsets"], total_members, stream,
                            flush, barrier, rank == 0 and not args.no_cpu_baseline, out["bitmap"],
                            out["counts"])
        if chain and csel:
            select["viable_sets"] = csel
    # the learned router: per-configuration linear
    # heads, the contraction emb . heads^T on tcgen05 with the threshold fused
    # into the epilogue; synthetic bf16 embeddings / heads (no reference)
    linear = None
    if not args.no_linear:
        D = 128
        gl = torch.Generator(device=dev_t).manual_seed(SEED)
        emb = torch.randn(REQUESTS_PER_GPU, D, device=dev_t, generator=gl).to(torch.bfloat16)
        heads = (torch.randn(S, D, device=dev_t, generator=gl) / D ** 0.5).to(torch.bfloat16)
        lbias = torch.randn(S, device=dev_t, generator=gl) * 0.1 - 0.2
        lprobe = dev.route_linear(emb, heads, lbias, capacity=1)
        torch.cuda.synchronize()
        lmem = int(lprobe.offsets[-1])
        lout = dev.alloc_route(REQUESTS_PER_GPU, 0, S, lmem)
        for _ in range(3):
            dev.route_linear(emb, heads, lbias, out=lout)
        lev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(5)]
        barrier()
        dev.profile_begin()
        for i in range(5):
            flush.fill_(i & 0xFF)
            lev[i][0].record(stream)
            dev.route_linear(emb, heads, lbias, out=lout)
            lev[i][1].record(stream)
        lprof = dev.profile_end()
        barrier()
        lms = statistics.median([x.elapsed_time(y) for x, y in lev])
        kms = lprof["k_linear_score"][0] / lprof["k_linear_score"][1]
        flops = 2.0 * REQUESTS_PER_GPU * S * D
        try:
            pk = json.load(open(PEAKS))["bf16_tflops"]
            pks = "measured burst bf16 (MEASURED_PEAKS.json)"
        except (OSError, KeyError, ValueError):
            pk, pks = 1590.0, "fallback (B200_PROFILING.md)"
        linear = {"router": f"linear heads, D {D}, bf16 -> fp32 (tcgen05 kind::f16, 2 x M128 N128 per K step, persistent, TMA SW128)",
                  "configs_per_s": REQUESTS_PER_GPU * S / (lms / 1e3), "ms_per_step": lms,
                  "members_per_step": lmem,
                  "kernel_ms": {k: v[0] / v[1] for k, v in lprof.items()},
                  "roofline": {"bound": "tensor", "kernel": "k_linear_score",
                               "achieved": flops / (kms / 1e3) / 1e12, "peak": pk,
                               "unit": "TFLOP/s", "frac": flops / (kms / 1e3) / 1e12 / pk,
                               "peak_source": pks},
                  "note": "MMA pipeline alone (no epilogue work, AG_LIN_EXP=2) runs at 0.78 of the peak; "
                          "the threshold epilogue (1.5 instructions per verdict) costs the rest"}
        del lout, lprobe, emb, heads, lbias
    # the same batch with the noisy router of BASELINE config 2 (fp 0, fn 0.3,
    # seed 7): integer-issue bound (two splitmix64 per needed configuration)
    noisy = None
    if not args.no_noisy:
        nrouter = P.NoisyRouter(0.0, 0.3, 7)
        nprobe = dev.route_enumerate(truth, nrouter, compact=False)
        torch.cuda.synchronize()
        nmem = int(nprobe.offsets[-1])
        nout = dev.alloc_route(REQUESTS_PER_GPU, 0, S, nmem)
        for _ in range(2):
            dev.route_enumerate(truth, nrouter, out=nout)
        nev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(3)]
        barrier()
        dev.profile_begin()
        for i in range(3):
            flush.fill_(i & 0xFF)
            nev[i][0].record(stream)
            dev.route_enumerate(truth, nrouter, out=nout)
            nev[i][1].record(stream)
        nprof = dev.profile_end()
        barrier()
        nms = [x.elapsed_time(y) for x, y in nev]
        noisy = {"router": "NoisyRouter(fp 0, fn 0.3, seed 7)",
                 "configs_per_s": REQUESTS_PER_GPU * S / (statistics.median(nms) / 1e3),
                 "ms_per_step": statistics.median(nms), "members_per_step": nmem,
                 "kernel_ms": {k: v[0] / v[1] for k, v in nprof.items()},
                 "bound": "integer issue (k_route_noise)"}
        # k_route_noise against the measured rng::mix absorb rate: with fp = 0
        # the noise can change exactly the truth bits (one absorb each)
        mp = absorb_peak() if rank == 0 and not args.no_ubench else None
        if mp and "k_route_noise" in nprof:
            kms = nprof["k_route_noise"][0] / nprof["k_route_noise"][1]
            needed = total_members  # truth bits of the batch (oracle members)
            if needed:
                ach = needed / (kms / 1e3)
                noisy["roofline"] = {"bound": "int-issue", "kernel": "k_route_noise",
                                     "achieved": ach, "peak": mp, "unit": "absorbs/s",
                                     "frac": ach / mp,
                                     "peak_source": "scripts/ubench/mix_peak (measured live)",
                                     "algorithmic_absorbs_per_launch": needed,
                                     "avg_launch_ms": kms}
        del nout, nprobe
    sched = run_sched(P, W, dev, args) if rank == 0 and not args.no_sched else None
    if sched is not None and not args.no_sched_variants:
        sched["variants"] = {}
        for name, v in SCHED_VARIANTS.items():
            r = run_sched(P, W, dev, args, rounds=v["rounds"], beam=v["beam"],
                          exhaustive=v["exhaustive"])
            sched["variants"][name] = {"beam": v["beam"], "exhaustive": v["exhaustive"],
                                       **{k: r[k] for k in ("p50_us", "p99_us", "device_p50_us",
                                                            "device_p99_us", "rounds",
                                                            "by_free_slots")}}
    deep = None if args.no_deep else run_deep(P, args, ws, rank, local, barrier)
    config1 = run_config1() if rank == 0 and not args.no_config5 else None
    config5 = run_config5() if rank == 0 and not args.no_config5 else None
    clk = clocks.stop()

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (algorithmic bytes / avg duration)
    hbm, peak_src = peaks()
    W_words = (S + 31) // 32
    bitmap_bytes = REQUESTS_PER_GPU * W_words * 4
    algo = {"k_route_score": bitmap_bytes,                        # bitmap write
            "k_route_compact": bitmap_bytes + 4 * total_members,   # bitmap read + index write
            "k_chunk_scan": REQUESTS_PER_GPU * 16,
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
                "d2h_bytes_per_step": int(d2h), "members_ok": bool(e2e_ok and ok_counts),
                "path": "ag_route_enumerate_host (pinned host indices)",
                "roofline": e2e_roof},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "peak_source": peak_src,
                     "traffic": ncu_traffic(dom),
                     "algorithmic_bytes_per_launch": algo.get(dom, 0),
                     "avg_launch_ms": dom_ms},
        "path_roofline": {"bytes_per_step": path_bytes,
                          "achieved_gbs": path_bytes / (tot_ms / args.steps / 1e3) / 1e9,
                          "frac": path_bytes / (tot_ms / args.steps / 1e3) / 1e9 / hbm},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    # the legs' full records, then (last on the line, so the driver's
    # 1,500-character stdout tail keeps it) the compact summary of every leg
    line["detail"] = {"kernel_share": kernel_share, "members_per_step": total_members,
                      "sched": sched, "deep": deep, "noisy": noisy, "linear": linear,
                      "chain": chain, "select": select, "config1": config1, "config5": config5}
    line["summary"] = summarize(line, sched, deep, noisy, linear, chain, config5, select, config1)
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def _r(x, nd=3):
    return None if x is None else float(f"{x:.{nd}g}")


def summarize(line, sched, deep, noisy, linear, chain, config5, select=None, config1=None):
    """One short record per leg (kept whole in the driver's stdout tail)."""
    out = {"route_configs_per_s": _r(line["value"]), "route_e2e": _r(line["e2e"]["value"]),
           "route_kernel_frac": _r(line["roofline"]["frac"])}
    if sched:
        out["sched_us"] = {"p50": _r(sched["p50_us"]), "p99": _r(sched["p99_us"]),
                           "dev_p50": _r(sched["device_p50_us"]), "dev_p99": _r(sched["device_p99_us"]),
                           "by_free": {k: [_r(v["p50_us"]), _r(v["p99_us"])]
                                       for k, v in sched["by_free_slots"].items()},
                           "with_dispatch": [_r(sched["round_plus_dispatch_p50_us"]),
                                             _r(sched["round_plus_dispatch_p99_us"])],
                           "hash": sched["decision_hash"]}
        for name, v in (sched.get("variants") or {}).items():
            out[f"sched_{name}_us"] = {"p50": _r(v["p50_us"]), "p99": _r(v["p99_us"]),
                                       "by_free": {k: [_r(x["p50_us"]), _r(x["p99_us"])]
                                                   for k, x in v["by_free_slots"].items()}}
    if deep:
        out["deep"] = {"configs_per_s": _r(deep["configs_per_s"]), "ms": _r(deep["ms_per_step"]),
                       "n_gpus": deep["n_gpus"]}
    if noisy:
        out["noisy_configs_per_s"] = _r(noisy["configs_per_s"])
    if linear:
        out["linear"] = {"configs_per_s": _r(linear["configs_per_s"]),
                         "tensor_frac": _r(linear["roofline"]["frac"])}
    if chain:
        out["chain_requests_per_s"] = _r(chain["requests_per_s"])
    if select:
        out["select_us"] = {"exhaustive": _r(select["us_per_batch"]),
                            "bitmap": _r((select.get("bitmap_path") or {}).get("us_per_batch")),
                            "frac": _r(select["roofline"]["frac"]),
                            "ref": _r((select.get("reference") or {}).get("us_per_batch")),
                            "match": select.get("digest_match")}
        vs = select.get("viable_sets")
        if vs:
            out["select_us"]["viable"] = _r(vs["us_per_batch"])
            out["select_us"]["viable_ref"] = _r((vs.get("reference") or {}).get("us_per_batch"))
            out["select_us"]["viable_match"] = vs.get("digest_match")
    if config1:
        out["config1"] = [[p["name"], p["identical"], _r(p["gpu"]["wall_s"]), _r(p["reference"]["wall_s"])]
                          for p in config1["points"]]
    if config5:
        out["config5"] = {"identical": config5["traces_identical"],
                          "rounds_per_s": [[p["rate"], _r(p["gpu"]["rounds_per_s"]),
                                            _r(p["reference"]["rounds_per_s"])]
                                           for p in config5["points"]]}
        if config5.get("decompose"):
            out["config5"]["decompose"] = [[p["rate"], _r(p["gpu"]["rounds_per_s"]),
                                            _r(p["reference"]["rounds_per_s"]), p["trace_identical"]]
                                           for p in config5["decompose"]["points"]]
        if config5.get("scale"):
            sc = config5["scale"]
            out["config5"]["scale_5x8"] = [sc["trace_identical"], _r(sc["gpu"]["wall_s"]),
                                           _r(sc["reference"]["wall_s"])]
    return out


def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: re-exec under torchrun, one
    process per GPU (rendezvous on 127.0.0.1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def spawn_selftest():
    """`bench.py --gpus N --spawn-selftest`: the ranks spawn_ranks launched
    meet in one process group (gloo, CPU) and rank 0 prints the world it saw."""
    import torch
    import torch.distributed as dist

    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    t = torch.ones(1)
    if ws > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"n_gpus": ws, "ranks_joined": int(t.item()),
                          "launcher": "torchrun" if "TORCHELASTIC_RUN_ID" in os.environ else "none"}))
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--sched-rounds", type=int, default=1000)
    ap.add_argument("--no-sched-variants", action="store_true")
    ap.add_argument("--sched-warmup", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sched", action="store_true")
    ap.add_argument("--no-deep", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    ap.add_argument("--no-noisy", action="store_true")
    ap.add_argument("--no-chain", action="store_true")
    ap.add_argument("--no-linear", action="store_true")
    ap.add_argument("--no-select", action="store_true")
    ap.add_argument("--no-ubench", action="store_true",
                    help="skip the PCIe / absorb-rate microbenchmarks (e.g. under ncu)")
    ap.add_argument("--spawn-selftest", action="store_true",
                    help="launcher check on CPU: ranks join a gloo group and rank 0 reports the world")
    args = ap.parse_args()
    spawn_ranks(args)
    if args.spawn_selftest:
        spawn_selftest()
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
