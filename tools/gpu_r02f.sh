# full GPU suite (new: paged KV, schedule dump, multi-rank, sanitizer) + default bench + RSA select A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02f_pytest.txt 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/r02f_pytest.txt | tail -15
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02f_bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), d['ms_per_step'], d['roofline']['call'], round(d['roofline']['frac'],3), d['mufu_measured'])
print({k:(round(v['tflops'],1)) for k,v in d['per_call'].items()})
for k,v in d['configs'].items(): print(k, round(v['value'],2), round(v['us_per_step'],1), v['roofline']['bound'], v['roofline']['frac'], {c:round(x['ms'],4) for c,x in v['per_call'].items()})
"
FL_EXTRA="-DFL_SEL_WG=2" timeout 900 python -c "from paper_2511_02043_b200 import build as b; b.build()" > /dev/null 2>&1
timeout 600 python bench.py --variant rsa --steps 10 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/r02f_sel2.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/r02f_sel2.json').read().strip().splitlines()[-1]); print('SEL_WG=2', {k:round(v['ms'],4) for k,v in d['per_call'].items()})"
