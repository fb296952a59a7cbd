# ncu --set full of one kernel launch per variant in $NCU_VARIANTS; exports raw + source CSVs on the
# box (the .ncu-rep files are too big to bring back several at a time) and keeps the report only if KEEP_REP=1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in ${NCU_VARIANTS:-causal}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-attn_tc} -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-1} -o /tmp/prof_$v -f python bench.py --variant $v --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ncu_full_$v.log 2>&1; echo "ncu full $v rc=$?"
ncu -i /tmp/prof_$v.ncu-rep --page raw --csv > gpurun_out/prof_${v}_raw.csv 2>/dev/null
ncu -i /tmp/prof_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${v}_src.csv 2>/dev/null
gzip -f gpurun_out/prof_${v}_src.csv
if [ -n "$KEEP_REP" ]; then cp /tmp/prof_$v.ncu-rep gpurun_out/; fi
done
