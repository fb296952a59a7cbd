cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ipa.py -q -x 2>&1 | tail -2
python tools/experiments/ipa_err.py
cat > /tmp/ipa_time.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch
from paper_2511_02043_b200 import synth, fl
x = {k: v.cuda() for k, v in synth.ipa_inputs(384, seed=1).items()}
for _ in range(3): fl.ipa_fwd(**x)
torch.cuda.synchronize()
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ipa_launches.csv python /tmp/ipa_time.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ipa_launches.csv')))
h=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]; hdr=rows[h]
for r in rows[h+1:][-12:]:
    d=dict(zip(hdr,r)); print(d.get('Kernel Name','')[:60], d.get('Metric Value'))
PY
timeout 600 python tools/paper_grid.py --block-only 2>&1 | grep "ipa"
