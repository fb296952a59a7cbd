# guard-band tests, then the FL_TIMING per-phase breakdown of the small-head and headline kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_guard.py -q > gpurun_out/r02o_guard.txt 2>&1; echo "guard rc=$?"; tail -15 gpurun_out/r02o_guard.txt
PROBE_VARIANTS="evo_row evo_col softcap causal" bash tools/gpu_timing.sh
