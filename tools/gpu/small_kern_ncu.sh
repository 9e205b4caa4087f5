# ncu --set full of one ax_kernel and one topk_local_kernel launch inside fits at the 8-GPU shard shape
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --snps 125000 --steps 1 --warmup 3 --no-cpu"
timeout 300 $CMD > /dev/null 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ax_kernel -s 40 -c 2 -o gpurun_out/ax_s8 $CMD > gpurun_out/ax_ncu.log 2>&1; echo "ax rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:topk_local -s 20 -c 1 -o gpurun_out/topk_s8 $CMD > gpurun_out/topk_ncu.log 2>&1; echo "topk rc=$?"
