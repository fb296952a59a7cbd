#!/bin/bash
# backward: mask-free fast path for the P loop
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_evoformer_block.py -q 2>&1 | tail -2
for v in bwd_causal bwd_vanilla bwd_diff; do
timeout 300 python bench.py --variant $v --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03k_$v.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r03k_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],2))"
done
