#!/bin/bash
# round-2 check: host-pipeline chunking (8), bench parity field
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err; echo bench rc=$?
timeout 300 python bench.py --variant evo_row --steps 5 --warmup 3 > gpurun_out/r02e_evo.json 2>> gpurun_out/r02e_bench.err; echo evo rc=$?
python - <<'P'
import json
for f in ("gpurun_out/r02e_bench.json","gpurun_out/r02e_evo.json"):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["value"], d.get("e2e",{}).get("value"), json.dumps(d.get("parity")))
P
