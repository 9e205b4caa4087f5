cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fit.py -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --workload c2path --steps 3 --warmup 1 --no-cpu 2>&1 | tail -1 | cut -c1-400
timeout 900 python bench.py --workload c4cv --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/c4cv.json; cat gpurun_out/c4cv.json
