# per-phase cycle breakdown (FL_TIMING build) of the softmax warpgroups, plus the new parity tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "needle or leak or plant or fullsize or diff" > gpurun_out/r02b_pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02b_pytest.txt
FL_TIMING=1 python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > gpurun_out/r02b_timing_build.log 2>&1; echo "build rc=$?"
timeout 600 python tools/timing_probe.py causal softcap vanilla evo_row evo_col diff > gpurun_out/r02b_timing_probe.txt 2>&1; echo "probe rc=$?"
cat gpurun_out/r02b_timing_probe.txt
