# parity of every bf16 variant + bench of the flex variants
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.txt 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/pytest_parity.txt
for v in ${BENCH_VARIANTS:-alibi softcap causal vanilla}; do
  timeout 300 python bench.py --variant $v --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), 'ms', round(d['ms_per_step'],4), d['roofline']['frac'])" 2>/dev/null || tail -3 gpurun_out/bench_$v.err
done
