# launch lists of resident native fits at configs 1-2, warm caches (as in-stream)
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in c2 c1; do
  timeout 120 python tools/small_fits.py $c || exit 1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/small_${c}_warm.csv python tools/small_fits.py $c > /dev/null 2>&1
done
