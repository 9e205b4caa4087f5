# A/B of two builds of the library (_ab/old.so vs _ab/new.so): warm-cache launch
# lists of the config-3 bench and the 8-GPU shard shape, and the fit rates
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in old new old new; do
  cp _ab/$v.so paper_1608_01398_b200/libgenoiht_cuda.so
  timeout 300 python bench.py --snps 125000 --steps 20 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v shard', round(d['value'],1), 'it/s', round(d['ms_per_step'],3), 'ms/fit')"
done
for v in old new; do
  cp _ab/$v.so paper_1608_01398_b200/libgenoiht_cuda.so
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/topk_$v.csv -k regex:topk_local python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/topk_shard_$v.csv -k regex:topk_local python bench.py --snps 125000 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
done
cp _ab/new.so paper_1608_01398_b200/libgenoiht_cuda.so
