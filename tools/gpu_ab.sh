# A/B of FL_EXTRA builds (timing only): ABL_FLAGS is a |-separated list of flag sets
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
IFS='|' read -ra SETS <<< "${ABL_FLAGS}"
for fl in "" "${SETS[@]}"; do
  FL_EXTRA="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > gpurun_out/ab_build.log 2>&1 || { echo "build failed [$fl]"; tail -5 gpurun_out/ab_build.log; continue; }
  line="[$fl]"
  for v in ${BENCH_VARIANTS:-causal}; do
    timeout 300 python bench.py --variant $v --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
    r=$(python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print(round(d['value'],1))" 2>/dev/null || echo ERR)
    line="$line $v=$r"
  done
  echo "$line"
done
