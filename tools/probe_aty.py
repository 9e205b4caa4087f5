"""Quick X^T r throughput probe on a synthetic matrix (not the bench)."""
import argparse
import ctypes
import time

import numpy as np
import torch

import paper_1608_01398_b200 as gi
from paper_1608_01398_b200 import _native
from paper_1608_01398_b200._native import check, lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--p", type=int, default=1_000_000)
ap.add_argument("--miss", type=float, default=0.0)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--exact", action="store_true")
a = ap.parse_args()

t0 = time.time()
m = gi.PackedGenotypeMatrix.synthetic(a.n, a.p, seed=1608, missing_rate=a.miss)
torch.cuda.synchronize()
print(f"synth {a.n}x{a.p}: {time.time() - t0:.2f}s", flush=True)
npad = lib().gi_padded_samples(m.handle)
rng = np.random.default_rng(0)
r = torch.zeros(npad, dtype=torch.float32, device="cuda")
r[: a.n] = torch.as_tensor(rng.standard_normal(a.n), dtype=torch.float32)
rd = r.double()
srt = torch.tensor([float(r.double().sum())], dtype=torch.float64, device="cuda")
scal = torch.tensor([0.0, 0.0, float(r.double().sum()), 0.0], dtype=torch.float64, device="cuda")
g = torch.zeros(a.p, dtype=torch.float64, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = _native.ptr


def launch():
    if a.exact:
        check(lib().gi_dev_aty_exact(m.handle, None, None, P(rd), P(srt), 1.0, P(g), s))
    else:
        check(lib().gi_dev_aty_fast(m.handle, None, None, None, P(r), P(scal), 1.0, P(g), s))


for _ in range(3):
    launch()
torch.cuda.synchronize()
ev0 = torch.cuda.Event(enable_timing=True)
ev1 = torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(a.reps):
    ev0.record()
    launch()
    ev1.record()
    torch.cuda.synchronize()
    ts.append(ev0.elapsed_time(ev1))
nb = (a.n + 3) // 4
bytes_x = a.p * nb
ms = float(np.median(ts))
print(f"aty {'exact' if a.exact else 'fast'}: median {ms:.3f} ms  min {min(ts):.3f} ms  "
      f"packed {bytes_x / ms / 1e6:.1f} GB/s  (best {bytes_x / min(ts) / 1e6:.1f} GB/s)")
# correctness spot check vs exact kernel on a few SNPs
ref = torch.zeros_like(g)
check(lib().gi_dev_aty_exact(m.handle, None, None, P(rd), P(srt), 1.0, P(ref), s))
torch.cuda.synchronize()
err = (g - ref).abs().max().item() / max(ref.pow(2).mean().sqrt().item(), 1e-300)
print(f"max |fast-exact| / rms = {err:.3e}")
