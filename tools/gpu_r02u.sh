cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "evo or Evo or key_mask or gate or bias or small or schedule or guard" > gpurun_out/pytest_evo.txt 2>&1; echo "evo tests rc=$?"; tail -3 gpurun_out/pytest_evo.txt
bench() { for v in evo_row evo_col; do timeout 300 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$1 $v', round(d['value'],1), 'ms', round(d['ms_per_step'],4), d['roofline']['frac'])" 2>/dev/null || tail -3 gpurun_out/bench_$v.err; done; }
bench base
FL_EXTRA="-DFL_BIG" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > /dev/null 2>&1; bench bigq
FL_EXTRA="-DFL_BIG -DFL_BIG_NSLOT=12" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > /dev/null 2>&1; bench bigq12
