cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
GI_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --samples 20000 --snps 200000 2>&1 | tail -1 | cut -c1-300
timeout 600 python bench.py --no-cpu --steps 4 2>&1 | tail -1 | cut -c1-200
