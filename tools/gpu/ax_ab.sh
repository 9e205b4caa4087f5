# A/B of two library builds (_ab/old.so vs _ab/new.so): warm-cache ax_kernel
# launch lists at config 3, the 8-GPU shard shape and configs 1-2, then the tests
cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
for v in old new; do
  cp _ab/$v.so paper_1608_01398_b200/libgenoiht_cuda.so
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/ax_c3_$v.csv -k regex:ax_kernel python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/ax_shard_$v.csv -k regex:ax_kernel python bench.py --snps 125000 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
  for c in c1 c2; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/ax_${c}_$v.csv -k regex:ax_kernel python tools/small_fits.py $c > /dev/null 2>&1
  done
done
cp _ab/new.so paper_1608_01398_b200/libgenoiht_cuda.so
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
