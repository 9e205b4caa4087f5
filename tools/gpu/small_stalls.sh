# ncu --set full (source-level stalls) of one top-k and one X_S w launch at config 3
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:topk_local -s 40 -c 1 -o gpurun_out/prof_topk $CMD > gpurun_out/ncu_topk.log 2>&1; echo topk rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ax_kernel -s 60 -c 2 -o gpurun_out/prof_ax $CMD > gpurun_out/ncu_ax.log 2>&1; echo ax rc=$?
