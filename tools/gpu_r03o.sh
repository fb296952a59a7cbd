#!/bin/bash
# same-box A/B (gpurun_alt/libfl_attn_{base,pf}.so): Evoformer row attention
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for lib in base pf; do
cp gpurun_alt/libfl_attn_$lib.so paper_2511_02043_b200/libfl_attn.so
timeout 300 python bench.py --variant evo_row --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03o.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r03o.json').read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],4))"
done; done
cp gpurun_alt/libfl_attn_pf.so paper_2511_02043_b200/libfl_attn.so
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -k "evo" 2>&1 | tail -1
