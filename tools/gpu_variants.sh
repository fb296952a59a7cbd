# A/B experiment: rebuild on the box with each flag set in $FLAGSETS (";"-separated) and bench $BENCH_VARIANTS
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
IFS=';' read -ra SETS <<< "${FLAGSETS:-}"
for fs in "${SETS[@]}"; do
  FL_EXTRA="$fs" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > /tmp/b.log 2>&1 || { echo "build failed: $fs"; tail -5 /tmp/b.log; continue; }
  for v in ${BENCH_VARIANTS:-causal}; do
    timeout 300 python bench.py --variant $v --steps 10 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
    python -c "import json;d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]);print('[$fs]', '$v', round(d['value'],1), {k:(round(v.get('tflops',0),1)) for k,v in d['per_call'].items()})" 2>/dev/null || tail -3 /tmp/o.err
  done
done
