cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bwd.py -q -x 2>&1 | tail -4
for v in bwd_causal bwd_vanilla; do timeout 600 python bench.py --variant $v --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), 'ms', round(d['ms_per_step'],3))" 2>/dev/null || tail -3 gpurun_out/bench_$v.err; done
