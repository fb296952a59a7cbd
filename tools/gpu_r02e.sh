# A/B: softcap tanh polynomial, split-S, split-S+P; full GPU suite on the default build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$2', round(d['value'],1), 'ms', round(d['ms_per_step'],4), {k:(round(v.get('tflops',0),1), round(v['ms'],4)) for k,v in d['per_call'].items()}, 'clk', d['clocks'].get('sm_mhz'))" 2>&1 | tail -1; }
run_ab() {  # $1 = label, $2 = FL_EXTRA
  FL_EXTRA="$2" timeout 900 python -c "from paper_2511_02043_b200 import build as b; b.build()" > /dev/null 2>&1 || echo "build $1 failed"
  for v in flex diff vanilla evo_row; do
    timeout 600 python bench.py --variant $v --steps 10 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/r02e_$1_$v.json 2> gpurun_out/r02e_$1_$v.err; summ gpurun_out/r02e_$1_$v.json "$1 $v"
  done
}
run_ab base ""
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02e_pytest.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02e_pytest.txt
run_ab mufu "-DFL_SOFTCAP_MUFU"
run_ab splitS "-DFL_SPLIT"
run_ab splitSP "-DFL_SPLIT -DFL_SPLIT_P"
