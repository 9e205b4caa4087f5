# Config 5 after a missing-path change: bench line and full-size parity
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 1500 python bench.py --workload c5 --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 bench rc=$?"
timeout 900 python tools/parity_scale.py --n 500000 --p 20000 --k 100 --missing 0.02 --out gpurun_out/parity_c5slice.json 2>&1 | tail -1
timeout 2000 python tools/parity_scale.py --n 500000 --p 500000 --k 100 --missing 0.02 --out gpurun_out/parity_c5.json 2>&1 | tail -1
echo done
