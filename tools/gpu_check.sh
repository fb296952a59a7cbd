# usage: bash tools/gpu_check.sh <stage...>; every step under its own timeout
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { local t=$1; shift; local name=$1; shift; echo "== $name" ; timeout $t "$@" > gpurun_out/$name.txt 2>&1; echo "rc=$?" >> gpurun_out/$name.txt; tail -4 gpurun_out/$name.txt; }
for st in "$@"; do
case $st in
  smoke) run 90 smoke python __graft_entry__.py smoke ;;
  one) run 90 one python -m pytest tests/test_gpu_parity.py -q -x -k "vanilla_D128_S128" ;;
  bf16) run 900 bf16 python -m pytest tests/test_gpu_parity.py -q -k "bf16 or determinism or host or errors" ;;
  f32) run 400 f32 python -m pytest tests/test_gpu_parity.py -q -k "f32 or evoformer or diag" ;;
  gpu) run 1200 gpu python -m pytest tests -q -m gpu ;;
  bench) run 600 bench python bench.py ;;
esac
done
