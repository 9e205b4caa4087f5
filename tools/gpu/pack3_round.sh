# base-3 copy: GPU tests, stress, CV and C3 bench lines, pack3 kernel time
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 1200 python tools/stress_parity.py 200 90000 2>&1 | grep -v "^note" | tail -2
timeout 900 python tools/stress_cv.py 30 130000 2>&1 | tail -2
timeout 900 python bench.py --workload c4cv --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 s', d['cv_seconds'], d['k_best'])"
timeout 300 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['e2e']['value'], d['xtr_ms'], d['roofline']['frac'], d['clocks'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pack3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu 2>/dev/null | grep pack3 | cut -c1-400
