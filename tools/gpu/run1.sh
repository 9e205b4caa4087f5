set -x
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu 2>&1 | tail -25
timeout 120 python tools/probe_aty.py --n 100000 --p 100000 --reps 5 2>&1 | tail -5
timeout 300 python tools/probe_aty.py --n 100000 --p 1000000 --reps 10 2>&1 | tail -5
