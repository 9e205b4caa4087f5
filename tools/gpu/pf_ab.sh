# L2 prefetch distance A/B for X^T r (GI_XTR_PF blocks ahead of the TMA issuer)
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for pf in 0 1 2 4 0 2; do
GI_XTR_PF=$pf timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('b3 pf=$pf', round(d['value'],2), 'xtr_ms', round(d['xtr_ms'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
for pf in 0 2; do
GI_XTR_PF=$pf timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu --missing 0.02 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('miss pf=$pf', round(d['value'],2), 'xtr_ms', round(d['xtr_ms'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
