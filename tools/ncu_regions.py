#!/usr/bin/env python
"""Stall attribution by SASS region of an ncu source-page CSV: python tools/ncu_regions.py <src.csv[.gz]> [lo-hi ...]
Regions are hex address ranges (offsets within the function); prints samples and the stall-reason mix
per region, and the top instructions of each region."""
import csv, gzip, io, sys
path = sys.argv[1]
txt = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
rows = list(csv.reader(io.StringIO(txt)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
seen, uniq = set(), []
for r in data:
    if r[0] not in seen:
        seen.add(r[0]); uniq.append(r)
base = int(uniq[0][0], 16)
num = lambda x: float(x) if x.replace(".", "").isdigit() else 0.0
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_ex = hdr.index("Instructions Executed")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
regions = [(int(a, 16), int(b, 16)) for a, b in (x.split("-") for x in sys.argv[2:])] or [(0, 1 << 40)]
tot = sum(num(r[i_s]) for r in uniq)
for lo, hi_ in regions:
    rr = [r for r in uniq if lo <= int(r[0], 16) - base < hi_]
    s = sum(num(r[i_s]) for r in rr)
    ex = sum(num(r[i_ex]) for r in rr)
    mix = {h: sum(num(r[hdr.index(h)]) for r in rr) for h in stalls}
    mix = sorted(((v, k) for k, v in mix.items() if v), reverse=True)[:8]
    print(f"[{lo:#x},{hi_:#x}) samples {s:.0f} ({100*s/tot:.1f}%) warp-insts executed {ex:.0f}")
    print("   " + "  ".join(f"{k[6:]}={100*v/max(s,1):.0f}%" for v, k in mix))
    for r in sorted(rr, key=lambda r: -num(r[i_s]))[:12]:
        top = sorted(((num(r[hdr.index(h)]), h[6:]) for h in stalls), reverse=True)[:3]
        print(f"   {int(r[0],16)-base:#7x} {num(r[i_s]):6.0f} {r[1][:60]:60s} " + " ".join(f"{k}:{v:.0f}" for v, k in top if v))
