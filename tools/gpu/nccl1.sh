# NCCL backend on one GPU: world-of-one sharded loop (test + torchrun bench)
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -m gpu -x 2>&1 | tail -15
GI_FORCE_SHARDED=1 NCCL_DEBUG=WARN timeout 600 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 \
  --steps 4 --warmup 3 --no-cpu 2>&1 | tail -4
