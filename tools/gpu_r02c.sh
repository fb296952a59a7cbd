# ncu source-level profile of the causal kernel (softmax-warp stall attribution) + remaining new tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2511_02043_b200 import build as b; b.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x -k "needle or leak or plant or fullsize or diff or Diff" > gpurun_out/r02c_pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02c_pytest.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o /tmp/prof_causal -f python bench.py --variant causal --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-extra > gpurun_out/r02c_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_causal.ncu-rep --page raw --csv > gpurun_out/r02c_causal_raw.csv 2>/dev/null
ncu -i /tmp/prof_causal.ncu-rep --page source --csv --print-source sass > gpurun_out/r02c_causal_src.csv 2>/dev/null
gzip -f gpurun_out/r02c_causal_src.csv
ncu -i /tmp/prof_causal.ncu-rep --page details --csv > gpurun_out/r02c_causal_details.csv 2>/dev/null
timeout 600 python bench.py --steps 10 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/r02c_bench.json; tail -5 gpurun_out/r02c_bench.err
