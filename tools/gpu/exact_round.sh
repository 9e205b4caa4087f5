cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
echo "== fast kernel forced"; GI_XTR_EXACT=0 timeout 900 python -m pytest tests/test_gpu_fit.py tests/test_gpu_multirank.py -q -m gpu -x 2>&1 | tail -2
timeout 1200 python tools/stress_parity.py 400 90000 2>&1 | grep -v "^note" | tail -3
GI_XTR_EXACT=0 timeout 1200 python tools/stress_parity.py 200 90000 2>&1 | grep -v "^note" | tail -3
GI_LIB_PATH=$PWD/paper_1608_01398_b200/libgenoiht_cuda_debug.so timeout 600 python tools/sanitize_case.py 2>&1 | tail -1
timeout 300 python tools/lat_probe.py 2>&1 | grep "max_iter=200"
