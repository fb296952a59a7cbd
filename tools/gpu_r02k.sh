cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 120 python tools/bwd_debug.py 128 300 > gpurun_out/r02k_dbg.txt 2>&1; echo "dbg rc=$?"; head -c 1000 gpurun_out/r02k_dbg.txt
timeout -s KILL 900 python -m pytest tests/test_gpu_bwd.py -q -m gpu --timeout 300 > gpurun_out/r02k_bwd.txt 2>&1; echo "bwd rc=$?"; grep -E "passed|failed|FAILED|max-abs" gpurun_out/r02k_bwd.txt | head -40
timeout -s KILL 600 python bench.py --variant bwd_causal --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r02k_bench_bwd.json 2> gpurun_out/r02k_bench_bwd.err; echo "bench bwd rc=$?"; tail -c 1500 gpurun_out/r02k_bench_bwd.json; tail -3 gpurun_out/r02k_bench_bwd.err
timeout -s KILL 600 python bench.py --variant rsa --steps 10 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/r02k_rsa.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/r02k_rsa.json').read().strip().splitlines()[-1]); print('rsa', {k:round(v['ms'],4) for k,v in d['per_call'].items()})"
