"""Summarise an ncu --set full report into the profiles/*_ncu_full.json
layout: per launch (kernel name + a label per launch), the timing, DRAM
traffic, issue / occupancy and stall ratios.  usage:
python scripts/ncu_summary.py <report.ncu-rep> <out.json> [label ...]
(labels name the captured launches in order, e.g. the workload each ran)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "ns": 1e-3, "ms": 1e3}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    labels = sys.argv[3:]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    launches = []
    for i, r in enumerate(data):
        name = r[hdr.index("Kernel Name")]
        d = {"kernel": name, "label": labels[i] if i < len(labels) else ""}
        for k in KEYS:
            if k not in hdr:
                continue
            j = hdr.index(k)
            try:
                v = float(r[j].replace(",", ""))
            except ValueError:
                continue
            d[k] = v * SCALE.get(units[j], 1) if units[j] in SCALE else v
        launches.append(d)
    json.dump({"source": rep, "units": "bytes; gpu__time_duration in us", "launches": launches},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
