# decode A/B: GPU decode/RSA tests + rsa_decode bench for the default build, then each FL_EXTRA flag set
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -x -k "decode or rsa or short" > gpurun_out/pytest_decode.txt 2>&1; echo "decode tests rc=$?"; tail -2 gpurun_out/pytest_decode.txt
IFS='|' read -ra SETS <<< "${ABL_FLAGS}"
for rep in 1 2; do
for fl in "" "${SETS[@]}"; do
  FL_EXTRA="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > gpurun_out/ab_build.log 2>&1 || { echo "build failed [$fl]"; continue; }
  timeout 300 python bench.py --variant rsa_decode --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('[$fl]', 'step ms', round(d['ms_per_step'],4), {k:round(v['ms']*1000,1) for k,v in d['per_call'].items()}, 'frac', round(d['roofline']['frac'],3))" 2>/dev/null || echo "[$fl] ERR"
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > /dev/null 2>&1
