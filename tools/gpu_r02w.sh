cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
one() { timeout 300 python bench.py --variant softcap --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/b_sc.json 2> gpurun_out/b_sc.err; python -c "import json;d=json.loads(open('gpurun_out/b_sc.json').read().strip().splitlines()[-1]);print('$1 softcap', round(d['value'],1))" 2>/dev/null || tail -3 gpurun_out/b_sc.err; }
one base; one base2
for m in 0x01 0x11 0x49; do FL_EXTRA="-DFL_TANH_MUFU_MASK=$m" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > /dev/null 2>&1; one m$m; one m${m}b; done
