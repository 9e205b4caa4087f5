cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
GI_TRACE_FIT=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu 2>&1 | grep -E "gi_fit" | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu rc=$?
