cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in bwd_causal bwd_vanilla; do timeout 600 python bench.py --variant $v --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), 'ms', round(d['ms_per_step'],3), {k:(round(v.get('tflops',0),1), round(v['ms'],3)) for k,v in d['per_call'].items()})" 2>/dev/null || tail -3 gpurun_out/bench_$v.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:bwd -c 6 --csv --log-file gpurun_out/bwd_launches.csv python bench.py --variant bwd_causal --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/bwd_launches.csv')))
h=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
hdr=rows[h]
for r in rows[h+1:]:
    d=dict(zip(hdr,r)); print(d.get('Kernel Name','')[:40], d.get('Metric Name'), d.get('Metric Value'))
PY
