# measurement refresh: default bench line, launch list, ncu full of the changed kernels, paper grid
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02t_bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), {k:round(v['tflops'],1) for k,v in d['per_call'].items()}, d['roofline']['call'], round(d['roofline']['frac'],3), d['clocks'])
for c,e in d.get('configs',{}).items(): print(c, e.get('value'), e.get('unit'), {k:round(v['ms'],4) for k,v in e.get('per_call',{}).items()})
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 10 --csv --log-file gpurun_out/r02t_launches_flex.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-extra > /dev/null 2>&1; echo "ncu list rc=$?"
NCU_VARIANTS="softcap alibi evo_row" bash tools/gpu_prof.sh
timeout 900 python tools/paper_grid.py > gpurun_out/r02t_paper_grid.md 2> gpurun_out/r02t_paper_grid.err; echo "grid rc=$?"; tail -5 gpurun_out/r02t_paper_grid.err
