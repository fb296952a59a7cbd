#!/bin/bash
# ncu full capture of the IPA output kernel (source page for stalls)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ipa_out -c 1 -o gpurun_out/r03d_ipa_out python bench.py --variant ipa --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/r03d.log 2>&1; echo rc=$?
ncu -i gpurun_out/r03d_ipa_out.ncu-rep --page source --csv --print-source sass > gpurun_out/r03d_src.csv 2>/dev/null
ncu -i gpurun_out/r03d_ipa_out.ncu-rep --page details --csv > gpurun_out/r03d_details.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r03d_src.csv 25
grep -E "Duration|Registers|Achieved Occupancy|Theoretical Occupancy|Memory Throughput|DRAM Throughput|L1/TEX Hit|L2 Hit|Compute \(SM\) Throughput" gpurun_out/r03d_details.csv | head -20
