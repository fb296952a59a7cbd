cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 240 python -m pytest tests -q -m gpu -x -k "decode or rsa or short" > gpurun_out/pytest_decode.txt 2>&1; echo "decode tests rc=$?"; tail -4 gpurun_out/pytest_decode.txt
for v in ${BENCH_VARIANTS:-rsa_decode}; do
  timeout 300 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "$v rc=$?"; tail -3 gpurun_out/bench_$v.err | grep -i error; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],2), 'ms', round(d['ms_per_step'],4), {k:(round(v.get('tflops',0),1), round(v['ms'],4)) for k,v in d['per_call'].items()}, d['roofline']['frac'])" 2>/dev/null
done
