# quick iteration: parity (bf16 + f32) then causal bench + ncu full capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5
V=${1:-causal}
timeout 300 python bench.py --variant $V --no-cpu-baseline --no-e2e > gpurun_out/bench_$V.json 2>gpurun_out/bench_$V.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$V.json'));print(d['variant'] if 'variant' in d else '', round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['frac'], d['clocks'])"
if [ "$2" = prof ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/prof_$V -f python bench.py --variant $V --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
fi
