"""Aggregate ncu source-page stall samples per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv;
       python scripts/ncu_lines.py s.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.Counter(); text = {}
fname = ""; hdr = None; cur = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; iS = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) < len(hdr): continue
    if r[0].strip():
        cur = (fname, int(r[0])); text[cur] = r[1].strip()[:100]
    try: s = int(r[iS])
    except ValueError: continue
    if cur: agg[cur] += s
tot = sum(agg.values())
print("samples", tot)
for k, s in agg.most_common(top):
    print(f"{s:6d} {100*s/tot:5.1f}% {k[0]}:{k[1]}  {text.get(k,'')}")

# per-line stall breakdown for the top lines (set NCU_STALLS=1)
import os
if os.environ.get("NCU_STALLS"):
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    per = collections.defaultdict(collections.Counter)
    cur = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]; continue
        if not r or r[0] == "Line No" or len(r) < len(hdr): continue
        if r[0].strip(): cur = (fname, int(r[0]))
        for i in cols:
            try: per[cur][hdr[i]] += int(r[i])
            except ValueError: pass
    for k, s in agg.most_common(min(top, 8)):
        print(k, per[k].most_common(4))
