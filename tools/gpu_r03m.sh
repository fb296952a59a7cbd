#!/bin/bash
# same-box A/B of two prebuilt libraries (gpurun_alt/libfl_attn_{base,pf}.so), backward variants
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for lib in base pf; do
cp gpurun_alt/libfl_attn_$lib.so paper_2511_02043_b200/libfl_attn.so
for v in bwd_causal bwd_diff; do
timeout 300 python bench.py --variant $v --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03m.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r03m.json').read().strip().splitlines()[-1]); print('$lib', '$v', round(d['value'],1), round(d['ms_per_step'],2))"
done; done; done
