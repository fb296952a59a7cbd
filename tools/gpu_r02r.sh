cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/pytest_gpu.txt
bench() { for v in evo_row evo_col; do timeout 300 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]);print('$1 $v', round(d['value'],1), 'ms', round(d['ms_per_step'],4), d['roofline']['frac'])" 2>/dev/null || tail -3 gpurun_out/bench_$v.err; done; }
bench big
FL_EXTRA="-DFL_NO_BIG" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > /dev/null 2>&1; bench nobig
bench nobig2
