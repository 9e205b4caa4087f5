cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
make -s -C oracle >/dev/null 2>&1
timeout 900 python tools/parity_scale.py --n 100000 --p 1000000 --k 20 --out gpurun_out/parity_c3.json 2>&1 | tail -3
timeout 600 python tools/parity_scale.py --n 5000 --p 100000 --k 10 --out gpurun_out/parity_c2_k10.json 2>&1 | tail -1
timeout 600 python tools/parity_scale.py --n 5000 --p 100000 --k 50 --k-true 20 --out gpurun_out/parity_c2_k50.json 2>&1 | tail -1
timeout 900 python tools/parity_scale.py --n 500000 --p 20000 --k 100 --missing 0.02 --out gpurun_out/parity_c5slice.json 2>&1 | tail -1
timeout 1500 python tools/parity_scale.py --n 500000 --p 500000 --k 100 --missing 0.02 --out gpurun_out/parity_c5.json 2>&1 | tail -1
