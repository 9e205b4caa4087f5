cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x 2>&1 | tail -2
for v in 1 2; do echo "variant=$v"; GI_ATY_VARIANT=$v timeout 60 python tools/probe_aty.py --n 100000 --p 1000000 --reps 10 2>&1 | grep -E "aty fast|max"; done
for v in 1 2; do echo "variant=$v miss"; GI_ATY_VARIANT=$v timeout 60 python tools/probe_aty.py --n 500000 --p 100000 --miss 0.02 --reps 10 2>&1 | grep -E "aty fast|max"; done
