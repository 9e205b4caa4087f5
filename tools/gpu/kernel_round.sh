cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 1200 python tools/stress_parity.py 400 50000 2>&1 | tail -8
PYTHONPATH=$PWD:$PWD/oracle timeout 300 python tools/fast_err.py 2>&1 | tail -4
for miss in 0.0 0.02; do
timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu --missing $miss 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('missing $miss', round(d['value'],1), 'xtr_ms', round(d['xtr_ms'],3), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
