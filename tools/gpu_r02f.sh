#!/bin/bash
# diff backward: parity + bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --variant bwd_diff --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bwd_diff.json 2> gpurun_out/r02f.err; echo rc=$?
tail -3 gpurun_out/r02f.err
python -c "
import json
d=json.loads(open('gpurun_out/r02f_bwd_diff.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['gpu_launches'])"
