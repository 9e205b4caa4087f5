# one GPU's shard of config 3 on 8 GPUs (n = 100k, p = 125k): bench lines with and without the base-3 copy
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
for b in 1 0; do
GI_BASE3=$b timeout 300 python bench.py --snps 125000 --steps 20 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('base3=$b', round(d['value'],1), 'it/s', round(d['ms_per_step'],3), 'ms/fit xtr', round(d['xtr_ms'],4), 'ms frac', round(d['roofline']['frac'],3), d['iterations_per_fit'], d['clocks']['sm_mhz'])"
done
timeout 300 python tools/gap_probe.py 2>&1 | tail -4
