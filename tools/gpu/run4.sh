cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 120 python __graft_entry__.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fit.py -q -m gpu -x 2>&1 | tail -30
