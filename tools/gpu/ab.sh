# A/B of the native loop: _ab/ (previous build) vs the tree, same box
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fit.py -q -m gpu -x 2>&1 | tail -2
for r in 1 2; do
  echo "== prev"; GI_LIB_PATH=$PWD/_ab/libgenoiht_cuda.so timeout 300 python tools/lat_probe.py 2>&1 | grep "max_iter=200"
  echo "== new";  timeout 300 python tools/lat_probe.py 2>&1 | grep "max_iter=200"
done
