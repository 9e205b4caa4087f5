cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 300 python bench.py --snps 100000 --steps 3 --warmup 3 --cpu-slice 20000 2>&1 | tail -5
timeout 600 python bench.py 2>&1 | tail -5
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -3
