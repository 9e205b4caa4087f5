cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "fast or shapes" 2>&1 | tail -2
for f in 0 2 1; do echo "flags=$f"; GI_ATY_FLAGS=$f timeout 60 python tools/probe_aty.py --n 100000 --p 1000000 --reps 5 2>&1 | grep -E "aty fast|max"; done
