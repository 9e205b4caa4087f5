cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 900 python tools/stress_parity.py 200 80000 2>&1 | grep -v "^note" | tail -4
timeout 300 python tools/lat_probe.py 2>&1 | grep "max_iter=200"
for args in "" "--snps 125000" "--snps 250000"; do
timeout 300 python bench.py --no-cpu --steps 4 $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', '$args', round(d['value'],1), 'xtr_ms', round(d['xtr_ms'],4), 'GB/s', round(d['xtr_packed_gbs']), d['clocks']['sm_mhz'])"
done
timeout 300 python bench.py --workload c2path --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 path ms', round(d['ms_per_step'],2), d['parity'])"
