# bench + profile sequence (each step under its own timeout)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/bench_causal.json 2> gpurun_out/bench_causal.err; echo "causal rc=$?"; cat gpurun_out/bench_causal.json
for v in vanilla alibi sliding softcap document prefix gqa diff evo_row evo_col; do
  timeout 180 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "$v rc=$?"; cut -c1-400 gpurun_out/bench_$v.json
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_causal.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/prof_causal -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
