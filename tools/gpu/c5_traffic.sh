# ncu --set full of one config-5 X^T r launch -> profiles traffic record; then the c5 bench line
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
CMD="python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:aty_fast -s 5 -c 1 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"
python tools/traffic_json.py gpurun_out/prof_c5.ncu-rep --n 500000 --p 500000 --missing 0.02 --command "$CMD" --out profiles/aty_fast_traffic_c5.json
timeout 1500 python bench.py --workload c5 --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 bench rc=$?"
