#!/usr/bin/env python
"""Summarise ncu captures into the JSON/markdown kept under profiles/.

  python profiles/summarize_ncu.py full  <report.ncu-rep> <out.json>
  python profiles/summarize_ncu.py launches <launches.csv> <out.json>
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
       "lts__t_bytes.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def short(name):
    m = re.search(r"(k_[a-z_0-9]+)", name)
    return m.group(1) if m else name[:60]


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    # tensor-pipe counters (tcgen05 on sm_100a) wherever the capture has them
    extra = [h for h in hdr if h in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                                     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                                     "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                                     "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active")]
    metrics = RAW + extra
    agg = defaultdict(lambda: defaultdict(list))
    for r in data:
        k = short(r[col["Kernel Name"]])
        for m in metrics:
            if m in col:
                try:
                    agg[k][m].append(float(r[col[m]].replace(",", "")))
                except ValueError:
                    pass
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    unit_of = {h: u for h, u in zip(hdr, units)}
    for k, d in agg.items():
        for m in list(d):
            f = scale.get(unit_of.get(m, ""), 1.0)
            d[m] = [x * f for x in d[m]]
    res = {}
    for k, d in agg.items():
        e = {m: sum(v) / len(v) for m, v in d.items() if v}
        e["launches_captured"] = len(d.get("gpu__time_duration.sum", []))
        rd, wr = e.get("dram__bytes_read.sum"), e.get("dram__bytes_write.sum")
        if rd is not None and wr is not None:
            e["dram_bytes_per_launch"] = rd + wr
        res[k] = e
    json.dump({"source": rep, "units": "bytes; gpu__time_duration in us",
               "kernels": res}, open(out, "w"), indent=1, sort_keys=True)


def launches(path, out):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = defaultdict(lambda: [0.0, 0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        k = short(r["Kernel Name"])
        tot[k][0] += v
        tot[k][1] += 1
    all_us = sum(v[0] for v in tot.values())
    res = {k: {"total_us": v[0], "launches": v[1], "avg_us": v[0] / v[1], "share": v[0] / all_us}
           for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0])}
    json.dump({"source": path, "note": "cold-cache serialised ncu launch list; compare shares",
               "kernels": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
