# timing ablations (results wrong on purpose; timing only): FL_EXTRA builds, evo_row / evo_col bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for fl in "" ${ABL_FLAGS:-"-DFL_ABL_BIAS" "-DFL_ABL_KB" "-DFL_ABL_GATE"}; do
  FL_EXTRA="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > gpurun_out/abl_build.log 2>&1 || { echo "build failed $fl"; tail -5 gpurun_out/abl_build.log; continue; }
  for v in ${BENCH_VARIANTS:-evo_row evo_col}; do
    timeout 300 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/abl.json 2> gpurun_out/abl.err
    python -c "import json;d=json.loads(open('gpurun_out/abl.json').read().strip().splitlines()[-1]);print('[$fl] $v', round(d['ms_per_step'],4), 'ms')" 2>/dev/null || tail -3 gpurun_out/abl.err
  done
done
