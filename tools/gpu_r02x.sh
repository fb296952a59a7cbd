# full GPU tests + smoke + the default bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02x_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02x_pytest_gpu.txt
timeout 120 python __graft_entry__.py smoke > gpurun_out/r02x_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02x_smoke.txt
timeout 900 python bench.py > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err; echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02x_bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), {k:round(v['tflops'],1) for k,v in d['per_call'].items()}, d['roofline']['call'], round(d['roofline']['frac'],3), d['clocks'])
for c,e in d.get('configs',{}).items(): print(c, e.get('value'), e.get('unit'), {k:round(v['ms'],4) for k,v in e.get('per_call',{}).items()})
"
