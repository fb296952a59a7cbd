#!/bin/bash
# IPA finish split into a probabilities kernel (16 rows / CTA) and a per-row all-heads output kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ipa.py -q -x 2>&1 | tail -3
timeout 600 python tools/paper_grid.py --block-only 2>&1 | grep "| ipa"
timeout 300 python tools/experiments/ipa_err.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ipa --csv --log-file gpurun_out/r03c_ipa.csv python bench.py --variant ipa --steps 2 --warmup 1 --no-cpu-baseline --no-graph > /dev/null 2>&1
grep -v "^==" gpurun_out/r03c_ipa.csv | python -c "
import csv,sys
r=list(csv.DictReader(sys.stdin))
for x in r[-4:]: print(x['Kernel Name'][:40], x['Metric Name'], x['Metric Value'])"
