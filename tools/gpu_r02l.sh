cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_bwd.py -q -m gpu --timeout 300 > gpurun_out/r02l_bwd.txt 2>&1; echo "bwd rc=$?"; grep -E "passed|failed|^E " gpurun_out/r02l_bwd.txt | head -20
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_bwd_launches.csv python bench.py --variant bwd_causal --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu list rc=$?"
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/r02l_bwd_launches.csv')))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
h = rows[hi]; iname = h.index('Kernel Name'); iv = h.index('Metric Value')
for r in rows[hi+1:][-12:]:
    print(r[iname][:60], r[iv])
PY
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:bwd_dkdv -s 3 -c 1 -o /tmp/prof_dkdv -f python bench.py --variant bwd_causal --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/r02l_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_dkdv.ncu-rep --page source --csv --print-source sass > gpurun_out/r02l_dkdv_src.csv 2>/dev/null; gzip -f gpurun_out/r02l_dkdv_src.csv
ncu -i /tmp/prof_dkdv.ncu-rep --page raw --csv > gpurun_out/r02l_dkdv_raw.csv 2>/dev/null
