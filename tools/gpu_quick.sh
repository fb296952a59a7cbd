# parity + short bench of selected variants (env BENCH_VARIANTS), no ncu
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 700 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.txt
for v in ${BENCH_VARIANTS:-causal}; do
  timeout 180 python bench.py --variant $v --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "$v rc=$?"; tail -3 gpurun_out/bench_$v.err | grep -i error; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), 'ms', round(d['ms_per_step'],3), {k:(round(v.get('tflops',0),1), round(v['ms'],3)) for k,v in d['per_call'].items()})" 2>/dev/null
done
