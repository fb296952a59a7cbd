#!/bin/bash
# backward D = 64 (C3 bwd_diff): ncu full of one dK/dV and one dQ launch, stall tops
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in bwd_dkdv bwd_dq; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o /tmp/prof_$k -f python bench.py --variant ${BWD_V:-bwd_diff} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/r03j_$k.log 2>&1; echo rc=$?
ncu -i /tmp/prof_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r03j_${k}_src.csv 2>/dev/null
ncu -i /tmp/prof_$k.ncu-rep --page details --csv > gpurun_out/r03j_${k}_details.csv 2>/dev/null
echo "== $k"; python tools/ncu_stalls.py gpurun_out/r03j_${k}_src.csv 14
grep -o '"Duration","us","[0-9.]*"\|"Registers Per Thread","register/thread","[0-9]*"\|"Compute (SM) Throughput","%","[0-9.]*"\|"Memory Throughput","%","[0-9.]*"\|"Grid Size","","[0-9]*"' gpurun_out/r03j_${k}_details.csv
ncu -i /tmp/prof_$k.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[-1]
for key in ('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum'):
    if key in h: print(key, v[h.index(key)])"
done
