cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value'], 'xtr', d['xtr_ms'], 'ms/fit', d['ms_per_step'], 'launches', d['gpu_launches'])"
timeout 300 python bench.py --no-cpu --samples 5000 --snps 100000 --k 20 --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 value', d['value'], 'e2e', d['e2e']['value'], 'xtr', d['xtr_ms'], 'ms/fit', d['ms_per_step'], 'it/fit', d['iterations_per_fit'])"
timeout 300 python bench.py --no-cpu --samples 1000 --snps 10000 --k 10 --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 value', d['value'], 'e2e', d['e2e']['value'], 'xtr', d['xtr_ms'], 'ms/fit', d['ms_per_step'], 'it/fit', d['iterations_per_fit'])"
