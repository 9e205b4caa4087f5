cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
for ahead in 0 1 2 4 12; do echo "v2 ahead=$ahead"; GI_ATY_VARIANT=2 GI_ATY_L2AHEAD=$ahead timeout 60 python tools/probe_aty.py --n 100000 --p 1000000 --reps 10 2>&1 | grep -E "aty fast"; done
