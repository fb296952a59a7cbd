# split-tile MMA order: correctness (full GPU suite) + A/B against the unsplit order
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02d_pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02d_pytest.txt
summ() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$2', round(d['value'],1), 'ms', round(d['ms_per_step'],4), {k:(round(v.get('tflops',0),1), round(v['ms'],4)) for k,v in d['per_call'].items()}, 'frac', d['roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'))" 2>&1 | tail -1; }
for v in flex diff evo_row evo_col rsa vanilla; do
  timeout 600 python bench.py --variant $v --steps 10 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/r02d_split_$v.json 2> gpurun_out/r02d_split_$v.err; summ gpurun_out/r02d_split_$v.json "split $v"
done
FL_EXTRA="-DFL_NO_SPLIT" timeout 900 python -c "from paper_2511_02043_b200 import build as b; b.build()" > /dev/null 2>&1; echo "nosplit build rc=$?"
for v in flex diff evo_row evo_col rsa vanilla; do
  timeout 600 python bench.py --variant $v --steps 10 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/r02d_nosplit_$v.json 2> gpurun_out/r02d_nosplit_$v.err; summ gpurun_out/r02d_nosplit_$v.json "nosplit $v"
done
