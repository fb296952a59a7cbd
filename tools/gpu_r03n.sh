#!/bin/bash
# same-box A/B: fl_linear one CTA per SM (base) vs two (pf); Evoformer block bench + linear tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for lib in base pf; do
cp gpurun_alt/libfl_attn_$lib.so paper_2511_02043_b200/libfl_attn.so
timeout 300 python bench.py --variant evo_block --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03n.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r03n.json').read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],4))"
done; done
cp gpurun_alt/libfl_attn_pf.so paper_2511_02043_b200/libfl_attn.so
timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_evoformer_block.py -q 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:linear --csv --log-file gpurun_out/r03n_lin.csv python bench.py --variant evo_block --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
grep -v "^==" gpurun_out/r03n_lin.csv | python -c "
import csv,sys
for x in list(csv.DictReader(sys.stdin))[-3:]: print(x['Kernel Name'][:30], x['Metric Value'])"
