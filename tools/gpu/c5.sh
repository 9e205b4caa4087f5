cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
free -g | head -2
timeout 2400 python tools/parity_scale.py --n 500000 --p 500000 --k 100 --missing 0.02 --out gpurun_out/parity_c5.json > gpurun_out/c5.log 2>&1; echo rc=$?
tail -3 gpurun_out/c5.log
