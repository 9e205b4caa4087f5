cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 300 python tools/lat_probe.py 2>&1 | tail -10
