cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_bwd.py -q -m gpu --timeout 300 > gpurun_out/r02m_bwd.txt 2>&1; echo "bwd rc=$?"; grep -E "passed|failed|^E " gpurun_out/r02m_bwd.txt | head -20
for v in bwd_causal bwd_vanilla; do
timeout -s KILL 600 python bench.py --variant $v --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r02m_bench_$v.json 2> gpurun_out/r02m_bench_$v.err; echo "bench $v rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02m_bench_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), d['ms_per_step'])"
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_bwd_launches.csv python bench.py --variant bwd_causal --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu list rc=$?"
timeout -s KILL 1500 python tools/paper_grid.py > gpurun_out/r02m_paper_grid.md 2> gpurun_out/r02m_paper_grid.err; echo "grid rc=$?"; tail -5 gpurun_out/r02m_paper_grid.md; tail -3 gpurun_out/r02m_paper_grid.err
