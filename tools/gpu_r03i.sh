#!/bin/bash
# fl_linear bias staging: tests + evo_block bench + per-launch times
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_evoformer_block.py -q 2>&1 | tail -2
timeout 300 python bench.py --variant evo_block --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r03i_evo_block.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r03i_evo_block.json').read().strip().splitlines()[-1]); print('evo_block ms', d['ms_per_step'], d['per_call'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:linear --csv --log-file gpurun_out/r03i_lin.csv python bench.py --variant evo_block --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
grep -v "^==" gpurun_out/r03i_lin.csv | python -c "
import csv,sys
for x in list(csv.DictReader(sys.stdin))[-3:]: print(x['Kernel Name'][:30], x['Metric Value'])"
