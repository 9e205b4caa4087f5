# after a native-loop change: GPU tests, parity stress (single, CV), sanitizer, latency, C2 path
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 1200 python tools/stress_parity.py 400 90000 2>&1 | grep -v "^note" | tail -3
GI_STRESS_LARGE=1 timeout 900 python tools/stress_parity.py 30 70000 2>&1 | grep -v "^note" | tail -3
timeout 900 python tools/stress_cv.py 60 130000 2>&1 | tail -3
GI_LIB_PATH=$PWD/paper_1608_01398_b200/libgenoiht_cuda_debug.so timeout 600 python tools/sanitize_case.py 2>&1 | tail -1
timeout 300 python tools/lat_probe.py 2>&1 | grep "max_iter=200"
timeout 300 python bench.py --workload c2path --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 path ms', d['ms_per_step'], d['value'], d['parity'])"
timeout 900 python tools/stress_sharded.py 100 110000 2>&1 | tail -2
timeout 300 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['e2e']['value'], d['xtr_ms'], d['ms_per_step'], d['gpu_launches'], d['roofline']['frac'], d['clocks'])"
