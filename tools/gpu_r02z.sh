# round-2 final measurement pass: GPU tests, smoke, default bench, launch list, ncu full captures, paper grid, backward
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02z_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02z_pytest_gpu.txt
timeout 120 python __graft_entry__.py smoke > gpurun_out/r02z_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02z_smoke.txt
timeout 900 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err; echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02z_bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), {k:round(v['tflops'],1) for k,v in d['per_call'].items()}, d['roofline']['call'], round(d['roofline']['frac'],3), d['clocks'])
for c,e in d.get('configs',{}).items(): print(c, e.get('value'), e.get('unit'), {k:round(v['ms'],4) for k,v in e.get('per_call',{}).items()})
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 10 --csv --log-file gpurun_out/r02z_launches_flex.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-extra > /dev/null 2>&1; echo "ncu list rc=$?"
NCU_VARIANTS="softcap causal evo_row evo_col" bash tools/gpu_prof.sh
for v in bwd_causal bwd_vanilla; do timeout 600 python bench.py --variant $v --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02z_bench_$v.json 2>/dev/null; done
timeout 1200 python tools/paper_grid.py > gpurun_out/r02z_paper_grid.md 2> gpurun_out/r02z_paper_grid.err; echo "grid rc=$?"
