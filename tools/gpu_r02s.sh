cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/pytest_gpu.txt
flex() { timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/bench_flex_$1.json 2> gpurun_out/bench_flex_$1.err; python -c "import json,sys;d=json.loads(open('gpurun_out/bench_flex_$1.json').read().strip().splitlines()[-1]);print('$1 flex', round(d['value'],1), {k:round(v['tflops'],1) for k,v in d['per_call'].items()})" 2>/dev/null || tail -3 gpurun_out/bench_flex_$1.err; }
flex new
flex new2
FL_EXTRA="-DFL_ALIBI_FFMA" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > /dev/null 2>&1; flex alibi_ffma
