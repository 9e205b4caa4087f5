cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
for i in 1 2; do
echo "prev"; GI_LIB_PATH=$PWD/tools/libgenoiht_cuda_prev.so timeout 60 python tools/probe_aty.py --n 100000 --p 1000000 --reps 10 2>&1 | grep -E "aty fast"
echo "new"; timeout 60 python tools/probe_aty.py --n 100000 --p 1000000 --reps 10 2>&1 | grep -E "aty fast|max"
done
