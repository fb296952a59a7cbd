cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -k "rsa or sanitizer or paged or schedule or multirank or diff" > gpurun_out/r02g_pytest.txt 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|rror" gpurun_out/r02g_pytest.txt | tail -15
timeout 900 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/r02g_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r02g_bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), d['ms_per_step'], d['roofline']['call'], round(d['roofline']['frac'],3), d['mufu_measured'])
print({k:(round(v['tflops'],1)) for k,v in d['per_call'].items()})
for k,v in d['configs'].items(): print(k, round(v['value'],2), round(v['us_per_step'],1), v['roofline']['bound'], v['roofline']['frac'], {c:round(x['ms'],4) for c,x in v['per_call'].items()})
"
