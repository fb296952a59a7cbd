cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in evo_block ipa; do timeout 300 python bench.py --variant $v --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/b_$v.json 2> gpurun_out/b_$v.err; echo "$v rc=$?"; tail -c 600 gpurun_out/b_$v.json; tail -3 gpurun_out/b_$v.err; done
timeout 900 python bench.py > gpurun_out/r02aa_bench.json 2> gpurun_out/r02aa_bench.err; echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02aa_bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), d['clocks']); print(json.dumps(d.get('next')))"
tail -3 gpurun_out/r02aa_bench.err
