# round 2 first pass: GPU tests, every bench variant, Evoformer bias A/B (tensor-core identity add vs FFMA2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02a_gpu.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02a_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02a_pytest.txt
summ() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$2', round(d['value'],1), 'ms', round(d['ms_per_step'],4), {k:(round(v.get('tflops',0),1), round(v['ms'],4)) for k,v in d['per_call'].items()}, 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks'].get('sm_mhz'))" 2>&1 | tail -1; }
for v in flex diff evo_row evo_col rsa rsa_decode causal vanilla; do
  timeout 600 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/r02a_bench_$v.json 2> gpurun_out/r02a_bench_$v.err; echo "$v rc=$?"; summ gpurun_out/r02a_bench_$v.json $v
done
FL_EXTRA="-DFL_NO_BIAS_MMA" timeout 600 python -c "from paper_2511_02043_b200 import build as b; b.build()" > gpurun_out/r02a_build_ab.txt 2>&1; echo "ab build rc=$?"
for v in evo_row; do
  timeout 600 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/r02a_ab_$v.json 2> gpurun_out/r02a_ab_$v.err; echo "AB nobiasmma $v rc=$?"; summ gpurun_out/r02a_ab_$v.json $v
done
timeout 300 python -m pytest tests -q -m gpu -x -k "evo" > gpurun_out/r02a_ab_pytest.txt 2>&1; echo "ab evo pytest rc=$?"; tail -2 gpurun_out/r02a_ab_pytest.txt
