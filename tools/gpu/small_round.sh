# GPU tests, small-config latency, warm launch lists, C3 bench line
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 300 python tools/lat_probe.py 2>&1 | grep "max_iter=200"
for c in c2 c1; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/small_${c}_warm.csv python tools/small_fits.py $c > /dev/null 2>&1
done
timeout 300 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['e2e']['value'], d['xtr_ms'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['smem']['frac'], d['clocks'])"
timeout 300 python bench.py --workload c2path --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 path ms', d['ms_per_step'], d['value'], d['parity'])"
