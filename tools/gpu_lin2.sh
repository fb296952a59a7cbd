cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() {
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:linear --csv --log-file gpurun_out/lin_launches_$1.csv python bench.py --variant evo_block --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
python - "$1" <<'PY'
import csv, sys
rows=list(csv.reader(open(f'gpurun_out/lin_launches_{sys.argv[1]}.csv')))
h=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]; hdr=rows[h]
out={}
for r in rows[h+1:]:
    d=dict(zip(hdr,r)); out.setdefault((d['ID']), []).append((d['Metric Name'], d['Metric Value'], d.get('Grid Size')))
for k in list(out)[-3:]: print(sys.argv[1], out[k])
PY
}
run co


