# full bench + profile sequence (each step under its own timeout); results in gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_flex.json 2> gpurun_out/bench_flex.err; echo "flex rc=$?"; cut -c1-3000 gpurun_out/bench_flex.json
for v in ${BENCH_VARIANTS:-rsa rsa_decode diff evo_row evo_col causal vanilla gqa prefix}; do
  timeout 600 python bench.py --variant $v --steps 10 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "$v rc=$?"; tail -3 gpurun_out/bench_$v.err | grep -i error; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), 'ms', round(d['ms_per_step'],3), {k:(round(v.get('tflops',0),1), round(v['ms'],3)) for k,v in d['per_call'].items()}, 'e2e', round(d.get('e2e',{}).get('value',0),1), 'cpu', d.get('cpu_baseline',{}).get('value'))" 2>/dev/null
done
if [ -z "$NO_NCU" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 10 --csv --log-file gpurun_out/launches_flex.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu list flex rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 6 --csv --log-file gpurun_out/launches_rsa.csv python bench.py --variant rsa --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu list rsa rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 12 --csv --log-file gpurun_out/launches_rsa_decode.csv python bench.py --variant rsa_decode --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu list rsa_decode rc=$?"
NCU_VARIANTS="${NCU_VARIANTS:-causal softcap evo_row diff}" bash tools/gpu_prof.sh
NCU_VARIANTS="rsa" NCU_KERNEL="rsa_" NCU_SKIP=6 bash tools/gpu_prof.sh
fi
