"""Walker-only view of an ncu source capture of k_sched_round (diagnostics):
dynamic instructions and stall samples per source line of a file.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv;
       python scripts/ncu_walker.py s.csv [file] [steps] [top]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else "ag_sched_fast.cuh"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 64
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
hdr = None; fname = ""; cur = None
agg = collections.Counter(); ex = collections.Counter(); txt = {}; st = collections.Counter()
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]; continue
    if hdr is None or len(r) < len(hdr): continue
    if r[0].strip():
        cur = (fname, int(r[0])); txt[cur] = r[1].strip()[:80]
    try:
        s = int(r[iS]); e = int(r[iE] or 0)
    except ValueError:
        continue
    if cur:
        agg[cur] += s; ex[cur] += e
    if cur and cur[0] == want:
        for i in cols:
            try: st[hdr[i]] += int(r[i])
            except ValueError: pass
tot = sum(v for k, v in ex.items() if k[0] == want)
print(want, "dyn warp instr", tot, "per step", round(tot / steps, 1),
      "samples", sum(v for k, v in agg.items() if k[0] == want))
print(st.most_common(8))
for k, v in sorted(((k, v) for k, v in agg.items() if k[0] == want), key=lambda x: -x[1])[:top]:
    print(k[1], v, ex[k], txt.get(k))
