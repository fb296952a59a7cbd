#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_active.avg --clock-control none -k regex:decode --csv --log-file gpurun_out/r03a_dec.csv python bench.py --variant rsa_decode --steps 2 --warmup 1 --no-cpu-baseline --no-graph > /dev/null 2>&1; echo rc=$?
grep -v "^==" gpurun_out/r03a_dec.csv | python -c "
import csv,sys
r=list(csv.DictReader(sys.stdin))
for x in r[-6:]: print(x['Kernel Name'][:40], x['Metric Name'], x['Metric Value'])"
