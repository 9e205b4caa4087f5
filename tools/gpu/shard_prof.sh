cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/gpu/shard_shape.sh > gpurun_out/shard_shape.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/shard_launches.csv python tools/gap_probe.py > gpurun_out/shard_ncu.log 2>&1
echo rc=$?
