#!/usr/bin/env python
"""Top warp-stall SASS lines of an ncu source-page CSV (gzipped ok): python tools/ncu_stalls.py <src.csv[.gz]> [n] [ctx]"""
import csv, gzip, io, sys
path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
txt = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
rows = list(csv.reader(io.StringIO(txt)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
seen, uniq = set(), []
for r in data:
    if r[0] not in seen:
        seen.add(r[0]); uniq.append(r)
val = lambda r: int(r[i_s]) if r[i_s].isdigit() else 0
tot = sum(val(r) for r in uniq)
print(f"total samples {tot}, {len(uniq)} instructions")
order = sorted(range(len(uniq)), key=lambda i: -val(uniq[i]))[:n]
for i in order:
    if ctx:
        for r in uniq[max(0, i - ctx):i]:
            print(f"      {val(r):6d} {r[0][-5:]} {r[i_src][:90]}")
    r = uniq[i]
    print(f"{100*val(r)/tot:5.1f}% {val(r):6d} {r[0][-5:]} {r[i_src][:90]}")
    if ctx:
        print("   ---")
