# native loop under each speculation mode: GPU tests + small-config latency
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
for m in 0 2; do
  echo "== GI_FIT_SPEC=$m"
  GI_FIT_SPEC=$m timeout 900 python -m pytest tests/test_gpu_fit.py tests/test_gpu_reference_port.py -q -m gpu -x 2>&1 | tail -3
done
echo "== auto"
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python tools/lat_probe.py 2>&1 | tail -10
GI_TRACE_FIT=1 timeout 300 python tools/trace_fit.py 2>&1 | tail -4
