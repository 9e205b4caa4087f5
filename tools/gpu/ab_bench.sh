# A/B of bench shapes: _ab/ (library built from HEAD) vs the working tree
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
for args in "--snps 125000" "--snps 250000" "--samples 5000 --snps 100000"; do
  for lib in prev new; do
    if [ $lib = prev ]; then export GI_LIB_PATH=$PWD/_ab/libgenoiht_cuda.so; else unset GI_LIB_PATH; fi
    timeout 300 python bench.py --no-cpu --steps 6 $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$args', round(d['value'],1), 'xtr_ms', round(d['xtr_ms'],4), round(d['xtr_packed_gbs']), d['clocks']['sm_mhz'])"
  done
done
