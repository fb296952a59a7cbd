# round-2 closing measurement pass: smoke, default bench (all configs + next rows + parity), launch lists, decode ncu
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python __graft_entry__.py smoke > gpurun_out/r03z_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r03z_smoke.txt
timeout 1200 python bench.py > gpurun_out/r03z_bench.json 2> gpurun_out/r03z_bench.err; echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r03z_bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), {k:round(v['tflops'],1) for k,v in d['per_call'].items()}, d['roofline']['call'], round(d['roofline']['frac'],3), d['clocks'], 'e2e', round(d['e2e']['value'],1))
for c,e in d.get('configs',{}).items(): print(c, e.get('value'), e.get('unit'), {k:round(v['ms'],4) for k,v in e.get('per_call',{}).items()}, e['roofline'].get('frac'))
for c,e in d.get('next',{}).items(): print(c, e)
print(json.dumps(d.get('parity')))
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 10 --csv --log-file gpurun_out/r03z_launches_flex.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-extra > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r03z_launches_rsa_decode.csv python bench.py --variant rsa_decode --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu decode rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03z_launches_bwd_diff.csv python bench.py --variant bwd_diff --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu bwd_diff rc=$?"
