cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T() { timeout -s KILL "$@"; }
T 400 python -m pytest tests/test_gpu_rsa.py -q -m gpu -x --timeout 300 > gpurun_out/r02i_rsa.txt 2>&1; echo "rsa rc=$?"; tail -3 gpurun_out/r02i_rsa.txt
T 600 python -m pytest tests/test_gpu_bwd.py -q -m gpu --timeout 300 > gpurun_out/r02i_bwd.txt 2>&1; echo "bwd rc=$?"; grep -E "passed|failed|FAILED|max-abs" gpurun_out/r02i_bwd.txt | head -40
T 1200 python -m pytest tests -q -m gpu -x --timeout 600 -k "not sanitizer and not multirank and not test_gpu_rsa and not test_gpu_bwd" > gpurun_out/r02i_pytest.txt 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r02i_pytest.txt | tail -8
T 600 python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/r02i_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r02i_bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), d['ms_per_step'], d['roofline']['call'], round(d['roofline']['frac'],3), d['mufu_measured'])
print({k:(round(v['tflops'],1)) for k,v in d['per_call'].items()})
for k,v in d['configs'].items(): print(k, round(v['value'],2), round(v['us_per_step'],1), v['roofline']['bound'], v['roofline']['frac'], {c:round(x['ms'],4) for c,x in v['per_call'].items()})
"
T 1200 python -m pytest tests -q -m gpu --timeout 900 -k "sanitizer or multirank" > gpurun_out/r02i_pytest2.txt 2>&1; echo "pytest2 rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r02i_pytest2.txt | tail -8
