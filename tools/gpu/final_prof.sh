# Round-end evidence: default bench, reference arm, secondary workloads, the
# launch list of the default bench command and one ncu --set full of X^T r.
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --workload c2path > gpurun_out/bench_c2path.json 2>&1; echo "c2 rc=$?"
timeout 1200 python bench.py --workload c4cv > gpurun_out/bench_c4cv.json 2>&1; echo "c4 rc=$?"
timeout 1500 python bench.py --workload c5 --steps 3 > gpurun_out/bench_c5.json 2>&1; echo "c5 rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:aty_fast -s 5 -c 1 -o gpurun_out/prof_final $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
for c in c2 c1; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/small_${c}_warm.csv python tools/small_fits.py $c > /dev/null 2>&1
done
echo done
