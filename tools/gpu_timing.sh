cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
FL_TIMING=1 python -c "import sys; sys.path.insert(0,'.'); from paper_2511_02043_b200 import build; build.build()" > gpurun_out/timing_build.log 2>&1; echo "build rc=$?"
timeout 600 python tools/timing_probe.py ${PROBE_VARIANTS:-causal vanilla} > gpurun_out/timing_probe.txt 2>&1; echo "probe rc=$?"
tail -40 gpurun_out/timing_probe.txt
