# X^T r with 2% missing (2-bit tiles, every group takes the missing-sum lookups)
# and missing-free over the 2-bit tiles (GI_BASE3=0), plus the kernel tests
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu --missing 0.02 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('miss', round(d['value'],2), 'xtr_ms', round(d['xtr_ms'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
GI_BASE3=0 timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2bit', round(d['value'],2), 'xtr_ms', round(d['xtr_ms'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fit.py -q -m gpu -x 2>&1 | tail -2
