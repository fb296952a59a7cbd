cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_evoformer_block.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --variant evo_block --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/b_eb.json 2> gpurun_out/b_eb.err; python -c "import json;d=json.loads(open('gpurun_out/b_eb.json').read().strip().splitlines()[-1]);print('evo_block ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
cat > /tmp/lt.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch
from paper_2511_02043_b200 import bench_helpers if False else fl
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:linear --csv --log-file gpurun_out/lin_launches.csv python bench.py --variant evo_block --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/lin_launches.csv')))
h=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]; hdr=rows[h]
for r in rows[h+1:][-6:]:
    d=dict(zip(hdr,r)); print(d.get('Kernel Name','')[:40], d.get('Grid Size'), d.get('Metric Value'))
PY
