#!/bin/bash
# decode: warp-independent online softmax (no per-block barriers)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_paged.py tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -q -x -k "decode or short or paged or rsa or guard or sq" 2>&1 | tail -3
for i in 1 2; do
timeout 300 python bench.py --variant rsa_decode --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02h_dec.json 2> gpurun_out/r02h.err; echo rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/r02h_dec.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d['per_call']), d['roofline']['frac'])"
done
