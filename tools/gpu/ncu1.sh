cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
CMD="python tools/probe_aty.py --n 100000 --p 300000 --reps 3"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:aty_fast -s 2 -c 1 -o gpurun_out/prof_fast $CMD > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/plain.log; tail -5 gpurun_out/ncu.log
