cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu_decode.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 12 --csv --log-file gpurun_out/launches_rsa_decode.csv python bench.py --variant rsa_decode --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "ncu list rc=$?"
