# The sharded native loop over NCCL at world size 1 (its exchange steps run as
# real one-rank collectives) on config 3: bench line
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
GI_FORCE_SHARDED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29613 bench.py --no-cpu > gpurun_out/bench_nccl1.json 2> gpurun_out/bench_nccl1.err; echo rc=$?
tail -1 gpurun_out/bench_nccl1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['xtr_ms'], d['config']['parallelism'], d['clocks']['sm_mhz'])"
