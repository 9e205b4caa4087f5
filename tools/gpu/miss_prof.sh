# X^T r with 2% missing genotypes (every group takes the second-lookup path)
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --missing 0.02"
timeout 300 $CMD 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('miss', d['value'], d['xtr_ms'], d['roofline']['frac'], d['clocks'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:aty_fast -s 5 -c 1 -o gpurun_out/prof_miss python bench.py --steps 1 --warmup 3 --no-cpu --missing 0.02 > gpurun_out/ncu_miss.log 2>&1
echo "ncu rc=$?"
