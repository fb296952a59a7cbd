#!/bin/bash
# evo_row: ncu full with the CUDA source correlation (top stall source lines)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o /tmp/prof_evo -f python bench.py --variant evo_row --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/r03g.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_evo.ncu-rep --page source --csv --print-source cuda > gpurun_out/r03g_cuda_src.csv 2>/dev/null
ncu -i /tmp/prof_evo.ncu-rep --page source --csv --print-source sass > gpurun_out/r03g_sass_src.csv 2>/dev/null
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/r03g_cuda_src.csv')))
hi=[i for i,r in enumerate(rows) if r and ('Warp Stall Sampling (All Samples)' in r)]
print('header rows', hi[:3])
h=rows[hi[0]]; print(h[:12])
iS=h.index('Warp Stall Sampling (All Samples)')
data=[r for r in rows[hi[0]+1:] if len(r)==len(h)]
tot=sum(float(r[iS] or 0) for r in data)
top=sorted(data,key=lambda r:-float(r[iS] or 0))[:30]
for r in top: print(f"{100*float(r[iS])/tot:5.1f}% {r[0][:6]} {r[1][:150]}")
P
