cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rsa.py -q -x > gpurun_out/pytest_rsa.txt 2>&1; echo "rsa tests rc=$?"; tail -5 gpurun_out/pytest_rsa.txt
for v in ${BENCH_VARIANTS:-rsa}; do
  timeout 300 python bench.py --variant $v --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "$v rc=$?"; tail -3 gpurun_out/bench_$v.err | grep -i error; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), 'ms', round(d['ms_per_step'],3), {k:(round(v.get('tflops',0),1), round(v['ms'],3)) for k,v in d['per_call'].items()}, d['roofline'])" 2>/dev/null
done
