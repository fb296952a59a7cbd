cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
FL_DEBUG_HANG=1 timeout -s KILL 600 python -c "from paper_2511_02043_b200 import build as b; b.build()" > gpurun_out/r02j_build.txt 2>&1; echo "build rc=$?"
timeout -s KILL 120 python tools/bwd_debug.py 128 300 > gpurun_out/r02j_dbg.txt 2>&1; echo "dbg rc=$?"; head -c 3000 gpurun_out/r02j_dbg.txt
timeout -s KILL 120 python tools/bwd_debug.py 64 128 > gpurun_out/r02j_dbg2.txt 2>&1; echo "dbg2 rc=$?"; head -c 2000 gpurun_out/r02j_dbg2.txt
