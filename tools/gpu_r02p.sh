cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "evo or Evo or key_mask or gate or bias or small or schedule or guard" > gpurun_out/pytest_evo.txt 2>&1; echo "evo tests rc=$?"; tail -25 gpurun_out/pytest_evo.txt
for v in evo_row evo_col; do
  timeout 300 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "$v rc=$?"; tail -3 gpurun_out/bench_$v.err | grep -i error; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), 'ms', round(d['ms_per_step'],4), d['roofline']['frac'])" 2>/dev/null
done
PROBE_VARIANTS="evo_row" bash tools/gpu_timing.sh > /dev/null 2>&1; head -32 gpurun_out/timing_probe.txt
