cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/ipa_time.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch
from paper_2511_02043_b200 import synth, fl
x = {k: v.cuda() for k, v in synth.ipa_inputs(384, seed=1).items()}
for _ in range(2): fl.ipa_fwd(**x)
torch.cuda.synchronize()
PY
timeout 300 ncu --set full --import-source on -k regex:ipa_finish -c 1 -o /tmp/ipaf -f python /tmp/ipa_time.py > /dev/null 2>&1
ncu -i /tmp/ipaf.ncu-rep --page source --csv --print-source sass > gpurun_out/ipa_finish_src.csv 2>/dev/null
ncu -i /tmp/ipaf.ncu-rep --page raw --csv > gpurun_out/ipa_finish_raw.csv 2>/dev/null
gzip -f gpurun_out/ipa_finish_src.csv
