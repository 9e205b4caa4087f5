# Round-2 evidence: GPU suite, smoke, default bench (config 3, parity + CPU
# baseline), reference arm, config 5 / 2 / 4 lines, the launch list of the
# default bench command, one ncu --set full of the X^T r kernel, and the
# config-5 X^T r pair (missum_kernel + aty_fast_kernel over the base-3 copy).
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/ev
make -s -C oracle >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev/gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/ev/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err; echo "ref rc=$?"
timeout 1500 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/ev/bench_c5.json 2> gpurun_out/ev/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --workload c2path --steps 5 --warmup 2 > gpurun_out/ev/bench_c2path.json 2> gpurun_out/ev/bench_c2path.err; echo "c2 rc=$?"
timeout 1200 python bench.py --workload c4cv --steps 3 --warmup 2 > gpurun_out/ev/bench_c4cv.json 2> gpurun_out/ev/bench_c4cv.err; echo "c4 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-parity"
timeout 300 $CMD > gpurun_out/ev/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/ev/launches_c3.csv $CMD > gpurun_out/ev/ncu_list.log 2>&1
echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:aty_fast -s 5 -c 1 -o gpurun_out/ev/prof_c3 $CMD > gpurun_out/ev/ncu_full.log 2>&1
echo "full rc=$?"
C5="python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:"missum|aty_fast" -c 2 --csv --log-file gpurun_out/ev/c5_xtr_kernels.csv $C5 > gpurun_out/ev/ncu_c5.log 2>&1
echo "c5 ncu rc=$?"
echo done
