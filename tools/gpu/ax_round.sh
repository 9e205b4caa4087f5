# ax_kernel change: shard-shape bench line, small-config latency, ax launch times at the shard shape
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python bench.py --snps 125000 --steps 20 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shard', round(d['value'],1), 'it/s', round(d['ms_per_step'],3), 'ms/fit xtr', round(d['xtr_ms'],4), d['clocks']['sm_mhz'])"
timeout 300 python tools/lat_probe.py 2>&1 | grep "max_iter=200"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ax_kernel -s 20 -c 60 --csv python bench.py --snps 125000 --steps 1 --warmup 3 --no-cpu 2>/dev/null | grep gpu__time | python -c "
import sys,csv,collections
t=collections.defaultdict(list)
for r in csv.reader(sys.stdin):
    t[r[4][:18]].append(float(r[-1]))
for k,v in t.items(): print(k, len(v), 'avg us', round(sum(v)/len(v)/1000,2))"
