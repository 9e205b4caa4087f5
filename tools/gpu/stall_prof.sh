# ncu --set full of X^T r: base-3 copy (config 3) and 2-bit tiles with 2% missing
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:aty_fast -s 5 -c 1 -o gpurun_out/prof_b3 python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_b3.log 2>&1
echo "b3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:aty_fast -s 5 -c 1 -o gpurun_out/prof_miss2 python bench.py --steps 1 --warmup 3 --no-cpu --missing 0.02 > gpurun_out/ncu_miss2.log 2>&1
echo "miss rc=$?"
