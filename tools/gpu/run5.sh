cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python -m paper_1608_01398_b200 bench --synthetic 5000,100000 --path 10:50:1 --mode gpu,gpu+seq --repetitions 3 --out gpurun_out/c2cli 2>&1 | tail -2
