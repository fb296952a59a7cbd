#!/bin/bash
# fl_linear (q|k|v|g projection of the Evoformer block): ncu full + stall tops
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:linear_ln -c 1 -o /tmp/prof_lin -f python bench.py --variant evo_block --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/r03h.log 2>&1; echo rc=$?
ncu -i /tmp/prof_lin.ncu-rep --page source --csv --print-source sass > gpurun_out/r03h_src.csv 2>/dev/null
ncu -i /tmp/prof_lin.ncu-rep --page details --csv > gpurun_out/r03h_details.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r03h_src.csv 20
grep -o '"Duration","us","[0-9.]*"\|"Registers Per Thread","register/thread","[0-9]*"\|"Achieved Occupancy","%","[0-9.]*"\|"Compute (SM) Throughput","%","[0-9.]*"\|"Memory Throughput","%","[0-9.]*"\|"DRAM Throughput","%","[0-9.]*"\|"L2 Hit Rate","%","[0-9.]*"\|"Grid Size","","[0-9]*"' gpurun_out/r03h_details.csv
